"""Dev: run one fuzz batch (tests/corpus.py) on the GPU and list the pairs whose
outcome differs from the reference golden digests.  Usage: dbg_case.py W O"""
import json
import os
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import corpus  # noqa: E402
import paper_2203_15561_b200 as ga  # noqa: E402

W, O = int(sys.argv[1]), int(sys.argv[2])
gold = json.load(open("tests/golden/fuzz.json"))
for case, ((w, o, k, prio), pairs) in zip(gold["cases"], corpus.fuzz_cases(gold["seed"], gold["batches"])):
    if (w, o) != (W, O):
        continue
    got = [str(corpus.digest(x)) for x in ga.align_batch(pairs, ga.WindowConfig(window=w, overlap=o, k=k, priority=prio))]
    print((w, o, k, prio), "bad:", [q for q, (a, b) in enumerate(zip(got, case["digests"])) if a != b])
    break
