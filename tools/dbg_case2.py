"""Dev: window distances of one fuzz batch, GPU vs oracle, per pair."""
import json
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import corpus  # noqa: E402
from paper_2203_15561_b200._abi import PackedBatch  # noqa: E402
from paper_2203_15561_b200.engine import run_packed  # noqa: E402
from oracle import oracle  # noqa: E402

W, O = int(sys.argv[1]), int(sys.argv[2])
gold = json.load(open("tests/golden/fuzz.json"))
for case, ((w, o, k, prio), pairs) in zip(gold["cases"], corpus.fuzz_cases(gold["seed"], gold["batches"])):
    if (w, o) != (W, O):
        continue
    k = k or w
    b = PackedBatch.from_pairs(pairs)
    g = run_packed(b, w, o, k, prio)
    e = oracle.align_packed(b, w, o, k, prio)
    for q in range(b.n_pairs):
        a0, a1 = int(g.win_off[q]), int(g.win_off[q + 1]) if q + 1 < b.n_pairs else g.dists.shape[0]
        gd, ed = g.dists[a0:a1].tolist(), e.dists[a0:a1].tolist()
        print(q, "len", len(pairs[q][0]), len(pairs[q][1]), "res_eq", bool(g.results[q] == e.results[q]),
              "dists_eq", gd == ed)
        if gd != ed:
            print("  gpu", gd[:40]); print("  ora", ed[:40])
            print("  gpu res", g.results[q]); print("  ora res", e.results[q])
    break
