import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import corpus
from paper_2203_15561_b200._abi import PackedBatch
from paper_2203_15561_b200.engine import run_packed
from oracle import oracle
for b, ((w, o, k, prio), pairs) in enumerate(corpus.fuzz_cases(2024, 5)):
    if b != 4: continue
    batch = PackedBatch.from_pairs(pairs[:2])
    g = run_packed(batch, w, o, k or w, prio); e = oracle.align_packed(batch, w, o, k or w, prio)
    print(g.results, e.results, e.distances(0, len(pairs[0][0]), w, o), e.distances(1, len(pairs[1][0]), w, o))
