"""Dev: repeat the reference-golden fuzz corpus (and budget-1 batches) N times
on the GPU against the reference digests / the oracle; counts mismatching
batches."""
import json, os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import corpus
import paper_2203_15561_b200 as ga
from oracle import oracle
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gold = json.load(open("tests/golden/fuzz.json"))
bad = 0
for rep in range(reps):
    for case, ((w, o, k, prio), pairs) in zip(gold["cases"], corpus.fuzz_cases(gold["seed"], gold["batches"])):
        got = [str(corpus.digest(x)) for x in ga.align_batch(pairs, ga.WindowConfig(window=w, overlap=o, k=k, priority=prio))]
        if got != case["digests"]:
            bad += 1
            print("rep", rep, "cfg", (w, o, k, prio), "bad", [q for q in range(len(got)) if got[q] != case["digests"][q]], flush=True)
for (w, o) in ((32, 31), (64, 63), (16, 15), (8, 7)):
    for (cfg_, pairs) in corpus.fuzz_cases(7000 + w, 40, pairs_per_batch=24, max_len=1500):
        cfg = ga.WindowConfig(window=w, overlap=o, k=w, priority=cfg_[3])
        got = [corpus.outcome_key(x) for x in ga.align_batch(pairs, cfg)]
        exp = [corpus.outcome_key(x) for x in oracle.align_batch(pairs, cfg, threads=8)]
        if got != exp:
            bad += 1
            print("budget1", (w, o), "bad", flush=True)
print("bad batches", bad)
