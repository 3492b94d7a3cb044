"""Device-resident timing of the fused kernel (ncu target; dev tool).

    python tools/dev_kernel.py [config] [count] [reps]
Runs ga_align_batch_device `reps` times on one config's pairs (inputs already
in HBM) and prints the CUDA-event time per launch (W = GA_DEV_W, default 64,
O = 3W/8 or 24 at 64, k = GA_DEV_K, default W).  Knobs: GA_LANE_GROUPS (0/1: the 16-lane group kernel), GA_GROUP (lockstep group size),
GA_BLOCK, GA_WARPS_PER_SM (read by the library at each launch).
"""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15561_b200 import _abi, engine, sim  # noqa: E402


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    count = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    batch, _ = sim.config_pairs(cfg_id, count=count)
    n = batch.n_pairs
    L = engine.lib()
    ctx = engine.context(0)
    W = int(os.environ.get("GA_DEV_W", 64))
    O = 3 * W // 8 if W != 64 else 24
    cfg = _abi.make_config(W, O, int(os.environ.get("GA_DEV_K", W)), "MSID",
                           os.environ.get("GA_MODE", "improved"))
    host = _abi.PackedResults.allocate(batch, W, O)
    dev = torch.device("cuda:0")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    order = engine.lpt_order(batch.pat_len)
    d = [up(x) for x in (batch.codes, batch.pat_off, batch.pat_len, batch.txt_off, batch.txt_len,
                         order, host.ops_off, host.win_off)]
    res = torch.empty(n * 64, dtype=torch.uint8, device=dev)
    ops = torch.empty(host.ops.shape[0], dtype=torch.uint8, device=dev)
    dst = torch.empty(host.dists.shape[0], dtype=torch.uint8, device=dev)
    din = _abi.GaBatchIn(n, d[0].data_ptr(), int(batch.codes.shape[0]), d[1].data_ptr(),
                         d[2].data_ptr(), d[3].data_ptr(), d[4].data_ptr(), d[5].data_ptr())
    dout = _abi.GaBatchOut(res.data_ptr(), d[6].data_ptr(), ops.data_ptr(), host.n_ops,
                           d[7].data_ptr(), dst.data_ptr(), int(host.dists.shape[0]))
    if hasattr(L, "ga_debug_thread_stats"):
        z = np.zeros(18, np.uint64)
        L.ga_debug_thread_stats(z.ctypes.data_as(C.c_void_p), 1)
    st = torch.cuda.Stream(dev)
    times = []
    for it in range(reps):
        if hasattr(L, "ga_debug_thread_stats") and it == reps - 1:
            z = np.zeros(18, np.uint64)
            L.ga_debug_thread_stats(z.ctypes.data_as(C.c_void_p), 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        rc = L.ga_align_batch_device(ctx, C.byref(din), C.byref(cfg), C.byref(dout),
                                     C.c_void_p(st.cuda_stream))
        b.record(st)
        assert rc == 0, L.ga_last_error(ctx)
        st.synchronize()
        times.append(a.elapsed_time(b))
    r = res.cpu().numpy().view(_abi.RESULT_DTYPE)
    if hasattr(L, "ga_debug_pair_times") and n <= 262144:
        pt = np.zeros(4 * n, np.uint64)
        L.ga_debug_pair_times(pt.ctypes.data_as(C.c_void_p), n)
        t0 = pt[:n].min()
        st_ms = (pt[:n] - t0) / 1e6
        fin_ms = (pt[n:2 * n] - t0) / 1e6
        full = pt[2 * n:3 * n].astype(np.int64)
        ho = pt[3 * n:]
        ho_ms = np.where(ho > 0, (ho.astype(np.float64) - t0) / 1e6, np.nan)
        q = [0, 1, 10, 50, 90, 99, 100]
        print("pair start ms pct " + " ".join(f"{p}:{np.percentile(st_ms, p):.1f}" for p in q))
        print("pair finish ms pct " + " ".join(f"{p}:{np.percentile(fin_ms, p):.1f}" for p in q))
        print("full-tier windows per pair pct " + " ".join(f"{p}:{np.percentile(full, p):.0f}" for p in q))
        slow = np.argsort(-fin_ms)[:8]
        print("slowest pairs (id, finish ms, full-tier windows, taken from the hand-over list ms):",
              [(int(i), round(float(fin_ms[i]), 1), int(full[i]), round(float(ho_ms[i]), 1)) for i in slow])
        print("handed-over pairs", int(np.isfinite(ho_ms).sum()))
        np.savez_compressed(os.path.join("gpurun_out", f"pairtimes_r1_cfg{cfg_id}.npz"),
                            start=st_ms, fin=fin_ms, full=full, handover=ho_ms)
    if hasattr(L, "ga_debug_thread_stats"):
        st = np.zeros(18, np.uint64)
        L.ga_debug_thread_stats(st.ctypes.data_as(C.c_void_p), 1)
        st = st.astype(np.float64)  # the last launch only
        print(f"band steps/launch {st[0]:.0f} active lanes/step {st[1] / max(st[0], 1):.2f} "
              f"full-tier windows {st[2]:.0f} hand-overs {st[3]:.0f} "
              f"cycles/band step {st[4] / max(st[0], 1):.0f} full-tier cycles/step {st[5] / max(st[0], 1):.0f} "
              f"warps finish own pairs over {(st[7] - st[6]) / 1e6:.2f} ms; lane 0 band DC cycles/step "
              f"{st[8] / max(st[0], 1):.0f} band TB cycles/step {st[9] / max(st[0], 1):.0f}; full-tier DC "
              f"cycles/window {st[10] / max(st[2], 1):.0f} TB {st[11] / max(st[2], 1):.0f}; group window "
              f"set-up cycles/step {st[12] / max(st[0], 1):.0f}, traceback rounds/step {st[13] / max(st[0], 1):.1f}; "
              f"hand-over tail windows {st[14]:.0f}, DC {st[15] / max(st[14], 1):.0f} TB {st[16] / max(st[14], 1):.0f} "
              f"whole window {st[17] / max(st[14], 1):.0f} cycles")
    import hashlib
    dig = hashlib.md5(res.cpu().numpy().tobytes() + dst.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"results+dists md5 {dig}")
    print(f"config {cfg_id} n={n} ms/launch {[round(x, 2) for x in times]} "
          f"best {min(times):.2f} ({n / min(times) * 1e3 / 1e6:.3f} M aln/s) "
          f"status {np.bincount(r['status'], minlength=4).tolist()}", flush=True)


if __name__ == "__main__":
    main()
