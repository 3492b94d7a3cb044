"""Dev check: tools/_thread_model.so (genasm_thread.cuh on the host) vs the oracle.

    python tools/check_model.py
"""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2203_15561_b200 import _abi, sim  # noqa: E402
from oracle import oracle  # noqa: E402
import corpus  # noqa: E402

_SO = os.path.join(ROOT, "tools", "_thread_model.so")
_SRC = [os.path.join(ROOT, "tools", "thread_model.cpp"),
        os.path.join(ROOT, "paper_2203_15561_b200", "csrc", "genasm_thread.cuh")]
if not os.path.exists(_SO) or any(os.path.getmtime(f) > os.path.getmtime(_SO) for f in _SRC):
    import subprocess
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _SO, _SRC[0]], check=True)
M = C.CDLL(_SO)


def model(batch, w, o, k, prio):
    out = _abi.PackedResults.allocate(batch, w, o)
    cfg = _abi.make_config(w, o, k, prio)
    tiers = np.zeros(4, np.int64)
    rc = M.model_align_batch(C.byref(batch.struct()), C.byref(cfg), C.byref(out.struct()),
                             tiers.ctypes.data_as(C.c_void_p))
    assert rc == 0
    return out, tiers


def compare(batch, w, o, k, prio, tag):
    got, tiers = model(batch, w, o, k, prio)
    exp = oracle.align_packed(batch, w, o, k, prio, threads=os.cpu_count())
    bad = np.nonzero(got.results != exp.results)[0].tolist()
    for q in range(batch.n_pairs):
        if q in bad or exp.results["status"][q] != 0:
            continue
        if got.cigar(q) != exp.cigar(q):
            bad.append(q)
            continue
        a, b = int(exp.win_off[q]), _abi.num_windows(int(batch.pat_len[q]), w, o)
        if not np.array_equal(got.dists[a:a + b], exp.dists[a:a + b]):
            bad.append(q)
    print(f"{tag}: n={batch.n_pairs} tiers(band,full,n0,wide)={tiers[:4].tolist()} bad={len(bad)}"
          + (f" first={bad[:3]} got={got.results[bad[0]]} exp={exp.results[bad[0]]}" if bad else ""),
          flush=True)
    return not bad


def main():
    ok = True
    for cid, count in ((1, 2000), (2, 2000), (3, 200), (4, 200), (5, 1500)):
        batch, _ = sim.config_pairs(cid, count=count)
        ok &= compare(batch, 64, 24, 64, "MSID", f"config{cid}")
    batch, _ = sim.config_pairs(5, count=1500)
    for (w, o, k) in ((64, 24, 16), (64, 24, 8), (32, 12, 8), (32, 12, 32), (48, 18, 30),
                      (64, 0, 64), (16, 5, 16)):
        for prio in ("MSID", "DISM", "SMDI"):
            ok &= compare(batch, w, o, k, prio, f"config5 w={w} o={o} k={k} {prio}")
    for (w, o, k, prio), pairs in corpus.fuzz_cases(4242, 120, pairs_per_batch=24, max_len=400):
        if w > 64:
            continue
        k = w if k is None else k
        b = _abi.PackedBatch.from_pairs(pairs)
        ok &= compare(b, w, o, k, prio, f"fuzz w={w} o={o} k={k} {prio}")
    print("ALL OK" if ok else "MISMATCHES")


if __name__ == "__main__":
    main()
