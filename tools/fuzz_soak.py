"""Dev: a long randomized soak of the GPU path against the oracle (tests/corpus.py).
Usage: python tools/fuzz_soak.py SEED BATCHES [PAIRS_PER_BATCH] [MAX_LEN]"""
import os
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import corpus  # noqa: E402
import paper_2203_15561_b200 as ga  # noqa: E402
from oracle import oracle  # noqa: E402

seed, nb = int(sys.argv[1]), int(sys.argv[2])
ppb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
ml = int(sys.argv[4]) if len(sys.argv) > 4 else 700
bad = 0
for b, ((w, o, k, prio), pairs) in enumerate(corpus.fuzz_cases(seed, nb, pairs_per_batch=ppb, max_len=ml)):
    for mode in ("improved", "baseline") if b % 10 == 0 else ("improved",):
        cfg = ga.WindowConfig(window=w, overlap=o, k=k, priority=prio, mode=mode)
        got = [corpus.outcome_key(x) for x in ga.align_batch(pairs, cfg)]
        exp = [corpus.outcome_key(x) for x in oracle.align_batch(pairs, cfg, threads=os.cpu_count())]
        if got != exp:
            bad += 1
            q = next(i for i in range(len(got)) if got[i] != exp[i])
            print("MISMATCH batch", b, (w, o, k, prio, mode), "pair", q, flush=True)
print("batches", nb, "bad", bad)
