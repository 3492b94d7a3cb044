import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200._abi import PackedBatch
from paper_2203_15561_b200.engine import run_packed
b = PackedBatch.from_pairs([("ACGT","ACGT"),("ACGT","AGGT")])
g = run_packed(b, 32, 12, 32, "MSID"); print(g.results)
