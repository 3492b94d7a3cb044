"""Golden fixtures for mode="baseline" (the unimproved engine), made by the
REFERENCE in the build container:

    python tests/golden/make_baseline_golden.py

Output (committed): tests/golden/baseline.json -- per-pair outcome digests
(tests/corpus.py: cigar, cost, text_consumed, window_distances, rows_computed
and the three access counters) of `bitalign.window.align_batch(..., mode=
"baseline")` over a randomized corpus and the first 200 pairs of config 1.
"""

from __future__ import annotations

import json
import os
import sys
from multiprocessing import Pool

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(ROOT, "tests"))

from bitalign.window import WindowConfig, align_batch  # noqa: E402

import corpus  # noqa: E402

SEED, BATCHES, PER_BATCH, MAX_LEN = 31, 40, 8, 300


def _run(job):
    (w, o, k, prio), pairs = job
    cfg = WindowConfig(window=w, overlap=o, k=k, priority=prio, mode="baseline")
    return {"cfg": [w, o, k, prio], "digests": [str(corpus.digest(x)) for x in align_batch(pairs, cfg)]}


def main() -> None:
    jobs = list(corpus.fuzz_cases(SEED, BATCHES, pairs_per_batch=PER_BATCH, max_len=MAX_LEN))
    with Pool(os.cpu_count()) as pool:
        cases = pool.map(_run, jobs, chunksize=1)
    sys.path.insert(0, ROOT)
    from paper_2203_15561_b200 import sim  # the bit-exact recipe port (pinned by sim.json)
    from paper_2203_15561_b200._abi import PackedBatch  # noqa: F401
    batch, _ = sim.config_pairs(1, count=200)
    pairs = [(sim.codes_to_str(batch.codes[batch.pat_off[q]:batch.pat_off[q] + batch.pat_len[q]]),
              sim.codes_to_str(batch.codes[batch.txt_off[q]:batch.txt_off[q] + batch.txt_len[q]]))
             for q in range(batch.n_pairs)]
    chunks = [pairs[a:a + 25] for a in range(0, len(pairs), 25)]
    with Pool(os.cpu_count()) as pool:
        parts = pool.map(_run, [((64, 24, 64, "MSID"), c) for c in chunks])
    cfg1 = [d for part in parts for d in part["digests"]]
    with open(os.path.join(HERE, "baseline.json"), "w") as fh:
        json.dump({"seed": SEED, "batches": BATCHES, "pairs_per_batch": PER_BATCH,
                   "max_len": MAX_LEN, "cases": cases, "cfg1_first200": cfg1}, fh)
    print("wrote baseline.json", len(cases), len(cfg1))


if __name__ == "__main__":
    main()
