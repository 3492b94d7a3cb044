"""Run by tests/test_check_build.py in a subprocess with GA_SO pointing at the
GA_CHECK build (_genasm_check.so): the kernel's contract checks (PrunedAccess
on a table read outside the stored columns/levels, ops/dists/ring/region
bounds) over the bench shapes and a fuzz corpus, every result compared with
the oracle.  Prints one JSON line: violations, first violation, mismatches."""

from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import corpus  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2203_15561_b200 import _abi, engine, sim  # noqa: E402


def compare(batch, w, o, k, prio):
    got = engine.run_packed(batch, w, o, k, prio, device=0)
    exp = oracle.align_packed(batch, w, o, k, prio, threads=os.cpu_count() or 1)
    bad = int((got.results != exp.results).sum())
    for q in range(batch.n_pairs):
        if exp.results["status"][q] == 0 and got.cigar(q) != exp.cigar(q):
            bad += 1
    return bad + int(not np.array_equal(got.dists, exp.dists))


def main():
    L = engine.lib()
    assert hasattr(L, "ga_debug_check"), "GA_SO is not the GA_CHECK build"
    st = np.zeros(4, np.uint64)
    L.ga_debug_check(st.ctypes.data_as(C.c_void_p), 1)
    cases = []
    for cid, count, pts in ((1, 2000, [(64, 24, 64, "MSID")]), (2, 2000, [(64, 24, 64, "MSID")]),
                            (3, 1500, [(64, 24, 64, "MSID"), (64, 24, 32, "DISM")]),
                            (4, 40, [(64, 24, 64, "MSID")]),
                            (5, 600, [(64, 24, 16, "MSID"), (32, 12, 32, "SMDI"), (64, 0, 64, "MSID"),
                                      (48, 18, 30, "IDSM"), (32, 12, 8, "MSID")])):
        batch, _ = sim.config_pairs(cid, count=count)
        for p in pts:
            cases.append((f"config{cid} {p}", batch, p))
    import json as _json
    gold = _json.load(open(os.path.join(ROOT, "tests", "golden", "fuzz.json")))
    for n, ((w, o, k, prio), pairs) in enumerate(corpus.fuzz_cases(gold["seed"], gold["batches"])):
        if w <= 64:  # the reference-golden corpus (DESIGN 9: W=32 O=31 among them)
            cases.append((f"gold{n}", _abi.PackedBatch.from_pairs(pairs),
                          (w, o, w if k is None else k, prio)))
    for n, ((w, o, k, prio), pairs) in enumerate(corpus.fuzz_cases(5151, 60, pairs_per_batch=24,
                                                                 max_len=2500)):
        if w <= 64:
            cases.append((f"fuzz{n}", _abi.PackedBatch.from_pairs(pairs), (w, o, w if k is None else k, prio)))
    # windows at d_min = m = 64 (a run of 'N' or lowercase longer than W: the
    # full tier's last pass holds level 64 alone)
    import random
    rng = random.Random(64)
    deep = []
    for q in range(48):
        core = "".join(rng.choice("ACGT") for _ in range(rng.randrange(100, 600)))
        cut = rng.randrange(0, len(core))
        run = ("N" if q % 2 else "a") * rng.randrange(64, 200)
        p = core[:cut] + run + core[cut:]
        deep.append((p, corpus.noisy_copy(rng, core, 0.05)))
    for prio in ("MSID", "IDSM"):
        cases.append((f"deep {prio}", _abi.PackedBatch.from_pairs(deep), (64, 24, 64, prio)))
    # budget-1 windows (O = W - 1): one pattern symbol per window
    b1, _ = sim.config_pairs(5, count=200)
    for (w, o) in ((32, 31), (64, 63), (16, 15)):
        cases.append((f"budget1 w{w}", b1, (w, o, w, "MSID")))
    mismatches = []
    for tag, batch, (w, o, k, prio) in cases:
        if compare(batch, w, o, k, prio):
            mismatches.append(tag)
    L.ga_debug_check(st.ctypes.data_as(C.c_void_p), 0)
    first = int(st[0])
    print(json.dumps({"cases": len(cases), "violations": int(st[1]),
                      "first": {"code": first >> 32, "line": first & 0xffffffff,
                                "a": int(st[2]), "b": int(st[3])} if first else None,
                      "mismatches": mismatches}))


if __name__ == "__main__":
    main()
