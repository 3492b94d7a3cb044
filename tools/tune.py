"""Dev tool: device-timed kernel over a config subset under env knob settings.

    python tools/tune.py "GA_GROUP=8" "GA_GROUP=16;GA_SMEM_KB=100"
env: TUNE_CFG (3), TUNE_COUNT (20000), TUNE_WOK ("64,24,64")
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_15561_b200 import _abi, engine, sim  # noqa: E402

cfg_id = int(os.environ.get("TUNE_CFG", 3))
count = int(os.environ.get("TUNE_COUNT", 20000))
W, O, K = [int(x) for x in os.environ.get("TUNE_WOK", "64,24,64").split(",")]
batch, _ = sim.config_pairs(cfg_id, count=count)
L = engine.lib()
ctx = engine.context(0)
dev = torch.device("cuda", 0)
out = _abi.PackedResults.allocate(batch, W, O)


def td(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


bufs = [td(x) for x in (batch.codes, batch.pat_off, batch.pat_len, batch.txt_off, batch.txt_len,
                        engine.lpt_order(batch.pat_len), out.ops_off, out.win_off)]
res = torch.empty(batch.n_pairs * 64, dtype=torch.uint8, device=dev)
ops = torch.empty(out.ops.shape[0], dtype=torch.uint8, device=dev)
dst = torch.empty(out.dists.shape[0], dtype=torch.uint8, device=dev)
din = _abi.GaBatchIn(batch.n_pairs, bufs[0].data_ptr(), batch.codes.nbytes,
                     *[b.data_ptr() for b in bufs[1:6]])
dout = _abi.GaBatchOut(res.data_ptr(), bufs[6].data_ptr(), ops.data_ptr(), ops.shape[0],
                       bufs[7].data_ptr(), dst.data_ptr(), dst.shape[0])
cfg = _abi.make_config(W, O, K, "MSID")
st = torch.cuda.Stream(dev)
ref = None
grid = [dict(x.split("=") for x in s.split(";") if x) for s in sys.argv[1:]] or [{}]
for knobs in grid:
    for k_, v in knobs.items():
        os.environ[k_] = v

    def run():
        rc = L.ga_align_batch_device(ctx, C.byref(din), C.byref(cfg), C.byref(dout),
                                     C.c_void_p(st.cuda_stream))
        assert rc == 0, L.ga_last_error(ctx)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run()
    run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    r = res.cpu().numpy()
    same = ref is None or np.array_equal(r, ref)
    ref = r if ref is None else ref
    print(f"{knobs} {ms:.2f} ms  {batch.n_pairs / ms * 1e3:.0f} aln/s  same={same}", flush=True)
    for k_ in knobs:
        del os.environ[k_]
