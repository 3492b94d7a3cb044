"""Dev tool: first fuzz batches where the GPU disagrees with the oracle, with details."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import corpus  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2203_15561_b200._abi import PackedBatch  # noqa: E402
from paper_2203_15561_b200.engine import run_packed  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 2024
shown = 0
for b, ((w, o, k, prio), pairs) in enumerate(corpus.fuzz_cases(seed, 80)):
    kk = k if k is not None else w
    batch = PackedBatch.from_pairs(pairs)
    g = run_packed(batch, w, o, kk, prio)
    e = oracle.align_packed(batch, w, o, kk, prio)
    for q in range(batch.n_pairs):
        gs, es = g.results[q], e.results[q]
        gc = g.cigar(q) if gs["status"] == 0 else ""
        ec = e.cigar(q) if es["status"] == 0 else ""
        if gs != es or gc != ec:
            print(f"batch {b} W={w} O={o} k={kk} prio={prio} pair {q} |P|={len(pairs[q][0])} "
                  f"|T|={len(pairs[q][1])}")
            print("  gpu", gs, gc[:100])
            print("  orc", es, ec[:100])
            print("  dists gpu", g.distances(q, len(pairs[q][0]), w, o)[:20])
            print("  dists orc", e.distances(q, len(pairs[q][0]), w, o)[:20])
            shown += 1
            if shown >= 6:
                sys.exit(0)
print("done")
