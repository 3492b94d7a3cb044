import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200._abi import PackedBatch
from paper_2203_15561_b200.engine import run_packed
from oracle import oracle
cases = [("ACGT","ACGT"),("ACGT","AGGT"),("ACGTACGTAC","ACGTTCGTAC"),("ACGT",""),("A"*70,"A"*70),("ACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGT","ACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGT")]
b = PackedBatch.from_pairs(cases)
for w,o,k in [(64,24,64),(32,12,32),(100,30,100)]:
    g = run_packed(b, w, o, k, "MSID"); e = oracle.align_packed(b, w, o, k, "MSID")
    for q in range(b.n_pairs):
        print(w, q, "GPU", g.results[q], g.cigar(q)[:80] if g.results[q]["status"]==0 else "")
        print(w, q, "ORC", e.results[q], e.cigar(q)[:80] if e.results[q]["status"]==0 else "")
