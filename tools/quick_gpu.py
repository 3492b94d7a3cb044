"""Ad-hoc GPU timing of the C-ABI host path on config shapes (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2203_15561_b200 import sim
from paper_2203_15561_b200.engine import run_packed
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
count = int(sys.argv[2]) if len(sys.argv) > 2 else None
t = time.time(); batch, _ = sim.config_pairs(cfg_id, count=count); print("gen", time.time() - t, flush=True)
for it in range(3):
    t = time.time(); out = run_packed(batch, 64, 24, 64, "MSID"); dt = time.time() - t
    print(f"cfg{cfg_id} n={batch.n_pairs} host-path {dt*1e3:.1f} ms  {batch.n_pairs/dt:.0f} aln/s status={np.bincount(out.results['status'])}", flush=True)
