"""Dev: host packing throughput (ga_pack2) on config-3-sized input."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200 import engine  # noqa: E402

n = 2_784_704_044
codes = np.random.default_rng(1).integers(0, 4, n, dtype=np.uint8)
print("cores", os.cpu_count(), flush=True)
for _ in range(3):
    t = time.perf_counter()
    p = engine.pack2(codes)
    dt = time.perf_counter() - t
    print(f"ga_pack2 {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms)", flush=True)
