"""Sweep the host-buffer path (ga_align_batch) over GA_CHUNKS on config 3.

Prints one line per setting: wall time per call (bytes in / 2-bit in), so the
copy/kernel overlap can be tuned.  Usage: python tools/e2e_sweep.py [count]
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200 import _abi, engine, sim  # noqa: E402


def pinned(a):
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = np.frombuffer(np.ascontiguousarray(a).tobytes(), dtype=np.uint8)
    return t


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else None
    batch, _ = sim.config_pairs(3, count=count)
    n = batch.n_pairs
    L = engine.lib()
    ctx = engine.context(0)
    cfg = _abi.make_config(64, 24, 64, "MSID")
    out = _abi.PackedResults.allocate(batch, 64, 24, ops2=True)
    h = [pinned(x) for x in (batch.codes, batch.pat_off, batch.pat_len, batch.txt_off,
                             batch.txt_len, out.ops_off, out.win_off)]
    h_res = torch.empty(n * 64, dtype=torch.uint8, pin_memory=True)
    h_ops = torch.empty(out.ops.shape[0], dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(out.dists.shape[0], dtype=torch.uint8, pin_memory=True)
    pk = engine.pack2(batch.codes)
    h_pk = pinned(pk.data)
    bins = {
        "bytes": _abi.GaBatchIn(n, h[0].data_ptr(), int(batch.codes.shape[0]), h[1].data_ptr(),
                                h[2].data_ptr(), h[3].data_ptr(), h[4].data_ptr(), None),
        "packed": _abi.GaBatchIn(n, h_pk.data_ptr(), int(batch.codes.shape[0]), h[1].data_ptr(),
                                 h[2].data_ptr(), h[3].data_ptr(), h[4].data_ptr(), None, 1, 0,
                                 None),
    }
    bout = _abi.GaBatchOut(h_res.data_ptr(), h[5].data_ptr(), h_ops.data_ptr(), out.n_ops,
                           h[6].data_ptr(), h_dst.data_ptr(), int(h_dst.shape[0]), 1)
    plans = os.environ.get("SWEEP_PLAN")
    settings = plans.split(";") if plans else os.environ.get("SWEEP", "1,2,3,4,6,8").split(",")
    for chunks in settings:
        if plans:
            os.environ["GA_CHUNK_PLAN"] = chunks
        else:
            os.environ["GA_CHUNKS"] = chunks
        row = [f"chunks={chunks:>2}"]
        for name, bin_ in bins.items():
            ts = []
            for _ in range(4):
                t0 = time.perf_counter()
                rc = L.ga_align_batch(ctx, C.byref(bin_), C.byref(cfg), C.byref(bout))
                ts.append(time.perf_counter() - t0)
                assert rc == 0, L.ga_last_error(ctx)
            best = min(ts[1:])
            row.append(f"{name} {best * 1e3:7.1f} ms ({n / best / 1e6:.3f} M aln/s)")
        print("  ".join(row), flush=True)


if __name__ == "__main__":
    main()
