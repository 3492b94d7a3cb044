"""Dev: the W=32 O=31 golden fuzz batch, GPU vs oracle, per pair: where the
results first differ (window, distances around it, CIGAR position)."""
import json, os, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import corpus
from paper_2203_15561_b200 import _abi
from paper_2203_15561_b200.engine import run_packed
from oracle import oracle

gold = json.load(open("tests/golden/fuzz.json"))
for case, ((w, o, k, prio), pairs) in zip(gold["cases"], corpus.fuzz_cases(gold["seed"], gold["batches"])):
    if (w, o) != (32, 31):
        continue
    k = w if k is None else k
    b = _abi.PackedBatch.from_pairs(pairs)
    g = run_packed(b, w, o, k, prio, device=0)
    e = oracle.align_packed(b, w, o, k, prio, threads=4)
    for q in range(b.n_pairs):
        rg, re = g.results[q], e.results[q]
        nw = _abi.num_windows(int(b.pat_len[q]), w, o)
        dg = g.dists[g.win_off[q]:g.win_off[q] + nw]
        de = e.dists[e.win_off[q]:e.win_off[q] + nw]
        if rg.tobytes() == re.tobytes() and np.array_equal(dg, de) and g.cigar(q) == e.cigar(q):
            continue
        bad = np.nonzero(dg != de)[0]
        fw = int(bad[0]) if bad.size else -1
        cg, ce = g.cigar(q), e.cigar(q)
        cpos = next((i for i in range(min(len(cg), len(ce))) if cg[i] != ce[i]), min(len(cg), len(ce)))
        print(f"pair {q}: |P|={b.pat_len[q]} |T|={b.txt_len[q]} gpu={tuple(rg)} ora={tuple(re)}")
        print(f"   first window diff {fw} of {nw}: gpu {dg[max(0,fw-3):fw+4].tolist()} ora {de[max(0,fw-3):fw+4].tolist()}")
        print(f"   cigar diff at {cpos}: gpu {cg[max(0,cpos-5):cpos+10]} ora {ce[max(0,cpos-5):cpos+10]}")
    break

if os.environ.get("GA_SO", "").endswith("_val.so"):
    import ctypes as C
    from paper_2203_15561_b200 import engine
    L = engine.lib()
    out = np.zeros(8, np.uint64)
    L.ga_debug_dev_bad(out.ctypes.data_as(C.c_void_p))
    print("dev_bad:", out.tolist())
