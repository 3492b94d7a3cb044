#!/usr/bin/env python
"""Bench: windowed improved-GenASM alignment of BASELINE config 3 on B200.

One step = one pass of the hot path (fused GenASM-DC + GenASM-TB kernel)
over the rank's whole batch: 138,929 synthetic 10 kb PacBio-like pairs
(~15% error, `bitalign simulate --emit-pairs` recipe, seed 10003, generated
by the bit-exact C++ port of the reference simulator).

  value   alignments/s with inputs resident in HBM (C-ABI device call,
          CUDA events on the launching stream, max over ranks)
  e2e     same metric through the C-ABI with pinned HOST buffers: H2D of the
          packed pairs, kernel, D2H of records + CIGAR ops + window distances
  roofline  int32 ALU: algorithmic ops of the DC recurrence per launch /
          measured launch time vs the live-measured int32 ALU peak
  cpu_baseline  the C port of the reference path (oracle/) on this host's
          cores, bounded sample

Multi-GPU: `torchrun --nproc-per-node N bench.py --gpus N`; one process per
GPU, no collective on the data path (pairs are independent).  Default is
weak scaling (each rank aligns its own config-3-sized batch, rank r > 0 with
seed 10003 + 1000 r); --scaling strong splits the one 138,929-pair batch
longest-first across ranks.

`--impl reference` times the reference path's CPU implementation (the C
oracle port, all host threads) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "alignments/sec and GCUPS (10 kb reads)"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--count", type=int, default=None, help="pairs per rank (default: config)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(cfg_id, rank, world, scaling, count):
    """Packed pairs for this rank (+ a description)."""
    from paper_2203_15561_b200 import engine, sim
    r = sim.CONFIGS[cfg_id]
    n = count or r.count
    threads = max(1, (os.cpu_count() or 1) // max(1, world))
    if scaling == "weak" or world == 1:
        seed = r.seed + 1000 * rank
        ref = sim.make_reference(r.ref_len, seed)
        lens = r.read_len if r.read_len else sim.mixed_lengths(n, seed)
        batch, _ = sim.recipe_pairs(ref, n, lens, r.sub, r.ins, r.dele, seed, threads)
        return batch, seed
    batch, _ = sim.config_pairs(cfg_id, count=n, threads=threads)
    idx = engine.split_lpt(batch.pat_len, 64, 24, world)[rank]
    from paper_2203_15561_b200.engine import _subset
    return _subset(batch, idx), r.seed


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def cpu_reference(batch, sample, steps, warmup):
    """The reference path's CPU implementation: the C port in oracle/ (the
    reference itself is Python and cannot travel to the GPU box)."""
    from oracle import oracle
    from paper_2203_15561_b200.engine import _subset
    n = min(sample, batch.n_pairs)
    sub = _subset(batch, np.arange(n))
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        oracle.align_packed(sub, 64, 24, 64, "MSID", threads=threads)
        if it >= warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    return {"value": n * len(times) / total, "unit": "alignments/s", "cores": threads,
            "kind": "port", "seconds": total,
            "sample": f"first {n} pairs of the workload, oracle/genasm_oracle.c "
                      f"(C restatement of bitalign.window.align), {threads} threads"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    args = parse_args()
    rank, world, local_rank = env_rank()
    cfg_desc = (f"config{args.config}: BASELINE.json configs[{args.config - 1}] recipe, "
                "W=64 O=24 k=64 priority MSID")

    if args.impl == "reference":
        if rank != 0:
            return 0
        batch, seed = workload(args.config, 0, 1, "weak", args.count)
        cb = cpu_reference(batch, args.cpu_sample, max(1, args.steps), max(0, args.warmup))
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"],
                "unit": "alignments/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * cb["seconds"] / max(1, args.steps),
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "u64", "data": f"synthetic (bitalign simulate recipe, seed {seed})",
                "config": {"workload": cfg_desc, "pairs_per_step": min(args.cpu_sample,
                                                                       batch.n_pairs)},
                "cpu_baseline": {"value": cb["value"], "unit": cb["unit"], "cores": cb["cores"],
                                 "kind": cb["kind"], "sample": cb["sample"],
                                 "cpu_model": cpu_model()},
                "e2e": {"value": cb["value"], "unit": "alignments/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    from paper_2203_15561_b200 import _abi, engine
    from paper_2203_15561_b200._abi import PackedResults

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    t_gen = time.perf_counter()
    batch, seed = workload(args.config, rank, world, args.scaling, args.count)
    gen_s = time.perf_counter() - t_gen
    n = batch.n_pairs
    L = engine.lib()
    ctx = engine.context(local_rank)
    W, O, K, PRIO = 64, 24, 64, "MSID"
    cfg = _abi.make_config(W, O, K, PRIO)
    order = engine.lpt_order(batch.pat_len)

    # ---- device-resident inputs/outputs (torch owns the HBM) ----
    host_out = PackedResults.allocate(batch, W, O)
    to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    d_codes, d_po, d_pl = to_dev(batch.codes), to_dev(batch.pat_off), to_dev(batch.pat_len)
    d_to, d_tl, d_ord = to_dev(batch.txt_off), to_dev(batch.txt_len), to_dev(order)
    d_res = torch.empty(n * 64, dtype=torch.uint8, device=dev)
    d_oo, d_wo = to_dev(host_out.ops_off), to_dev(host_out.win_off)
    d_ops = torch.empty(host_out.ops.shape[0], dtype=torch.uint8, device=dev)
    d_dst = torch.empty(host_out.dists.shape[0], dtype=torch.uint8, device=dev)
    din = _abi.GaBatchIn(n, d_codes.data_ptr(), int(batch.codes.nbytes), d_po.data_ptr(),
                         d_pl.data_ptr(), d_to.data_ptr(), d_tl.data_ptr(), d_ord.data_ptr())
    dout = _abi.GaBatchOut(d_res.data_ptr(), d_oo.data_ptr(), d_ops.data_ptr(),
                           int(host_out.ops.shape[0]), d_wo.data_ptr(), d_dst.data_ptr(),
                           int(host_out.dists.shape[0]))
    stream = torch.cuda.Stream(dev)  # non-null handle: the kernel and the events share it

    def step():
        rc = L.ga_align_batch_device(ctx, C.byref(din), C.byref(cfg), C.byref(dout),
                                     C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(L.ga_last_error(ctx).decode())

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches = 0
    barrier()
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for s in range(args.steps):
        evs[s][0].record(stream)
        step()
        evs[s][1].record(stream)
        launches += int(L.ga_last_launch_count(ctx))
    t_all1.record(stream)
    barrier()
    clock_info = clocks.stop()
    total_ms = t_all0.elapsed_time(t_all1)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms_max = max_over_ranks(total_ms)
    pairs_all = sum_over_ranks(float(n))
    value = pairs_all * args.steps / (total_ms_max * 1e-3)

    # ---- e2e: the same call over pinned host buffers (H2D + kernel + D2H) ----
    def pinned_copy(a):
        t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
        t.numpy()[:] = np.frombuffer(np.ascontiguousarray(a).tobytes(), dtype=np.uint8)
        return t
    # Inputs: one code byte per symbol (what PackedBatch holds); outputs: the
    # result records, window distances and 2-bit ops (ga_batch_out.ops2, packed
    # on the device).  ga_align_batch pipelines chunks over three streams.
    ops2_out = PackedResults.allocate(batch, W, O, ops2=True)
    h_in = [pinned_copy(x) for x in (batch.codes, batch.pat_off, batch.pat_len, batch.txt_off,
                                     batch.txt_len, ops2_out.ops_off, ops2_out.win_off)]
    h_res = torch.empty(n * 64, dtype=torch.uint8, pin_memory=True)
    h_ops = torch.empty(ops2_out.ops.shape[0], dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(host_out.dists.shape[0], dtype=torch.uint8, pin_memory=True)
    hin = _abi.GaBatchIn(n, h_in[0].data_ptr(), int(batch.codes.shape[0]), h_in[1].data_ptr(),
                         h_in[2].data_ptr(), h_in[3].data_ptr(), h_in[4].data_ptr(), None)
    hout = _abi.GaBatchOut(h_res.data_ptr(), h_in[5].data_ptr(), h_ops.data_ptr(),
                           ops2_out.n_ops, h_in[6].data_ptr(), h_dst.data_ptr(),
                           int(h_dst.shape[0]), 1)
    # ga_align_batch copies the sequences, lengths, offsets and the LPT order
    h2d = int(h_in[0].shape[0]) + sum(int(t.shape[0]) for t in h_in[1:]) + 4 * n
    d2h = int(h_res.shape[0] + h_ops.shape[0] + h_dst.shape[0])

    def e2e_run(bin_, steps):
        def once():
            rc = L.ga_align_batch(ctx, C.byref(bin_), C.byref(cfg), C.byref(hout))
            if rc != 0:
                raise RuntimeError(L.ga_last_error(ctx).decode())
        once()  # warm the context's own buffers
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            once()
        return max_over_ranks(time.perf_counter() - t0)
    e2e_s = e2e_run(hin, args.e2e_steps)
    e2e_value = pairs_all * args.e2e_steps / e2e_s
    res_bytes = h_res.numpy().copy()
    # variant: sequences already held 2 bits per symbol on the host (ga_batch_in.packed2)
    packed = engine.pack2(batch.codes)
    h_pk = pinned_copy(packed.data)
    hin_pk = _abi.GaBatchIn(n, h_pk.data_ptr(), int(batch.codes.shape[0]), h_in[1].data_ptr(),
                            h_in[2].data_ptr(), h_in[3].data_ptr(), h_in[4].data_ptr(), None,
                            1, int(packed.exceptions.shape[0]),
                            packed.exceptions.ctypes.data if packed.exceptions.shape[0] else None)
    e2e_pk_s = e2e_run(hin_pk, args.e2e_steps)
    e2e_pk_value = pairs_all * args.e2e_steps / e2e_pk_s
    if not np.array_equal(res_bytes, h_res.numpy()):
        raise RuntimeError("packed-input and byte-input host runs disagree")
    # variant: byte codes in, the call packs each chunk on the host (GA_PACK_HOST)
    hin_hp = _abi.GaBatchIn(n, h_in[0].data_ptr(), int(batch.codes.shape[0]), h_in[1].data_ptr(),
                            h_in[2].data_ptr(), h_in[3].data_ptr(), h_in[4].data_ptr(), None,
                            _abi.GA_PACK_HOST)
    e2e_hp_s = e2e_run(hin_hp, args.e2e_steps)
    e2e_hp_value = pairs_all * args.e2e_steps / e2e_hp_s
    if not np.array_equal(res_bytes, h_res.numpy()):
        raise RuntimeError("packed-input and byte-input host runs disagree")
    h2d_pk = h2d - int(h_in[0].shape[0]) + int(h_pk.shape[0]) + 8 * int(packed.exceptions.shape[0])

    # device path and host path must agree exactly
    dev_res = d_res.cpu().numpy()
    if not np.array_equal(dev_res, h_res.numpy()):
        raise RuntimeError("device-resident and host-buffer runs disagree")
    res = h_res.numpy().view(_abi.RESULT_DTYPE)
    status_counts = np.bincount(res["status"], minlength=4).tolist()

    # ---- algorithmic work (from the outputs) and roofline ----
    from ctypes import Structure, c_int64

    class GaWork(Structure):
        _fields_ = [(f, c_int64) for f in ("windows", "entries", "alu_ops", "cells",
                                            "pattern_bases", "tb_steps")]
    L.ga_work_stats.argtypes = [C.POINTER(_abi.GaBatchIn), C.POINTER(_abi.GaConfig),
                                C.POINTER(_abi.GaBatchOut), C.c_int, C.POINTER(GaWork)]
    L.ga_work_stats.restype = None
    L.ga_bench_alu_peak.argtypes = [C.c_int, C.c_int]
    L.ga_bench_alu_peak.restype = C.c_double
    work = GaWork()
    L.ga_work_stats(C.byref(hin), C.byref(cfg), C.byref(hout), os.cpu_count() or 1,
                    C.byref(work))
    avg_launch_s = statistics.mean(step_ms) * 1e-3
    achieved = work.alu_ops / avg_launch_s / 1e9
    peak = L.ga_bench_alu_peak(local_rank, 5) / 1e9
    cells_all = sum_over_ranks(float(work.cells))
    gcups = cells_all * args.steps / (total_ms_max * 1e-3) / 1e9
    bases_all = sum_over_ranks(float(work.pattern_bases))

    traffic_gb = None  # from the committed ncu capture of this kernel on this workload
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "ncu_traffic.json")) as f:
            traffic_gb = json.load(f)["dram_total_GB"]
    except (OSError, ValueError, KeyError):
        pass
    hbm = None  # the same traffic against the driver-measured HBM copy bandwidth
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                               "MEASURED_PEAKS.json")) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
        if traffic_gb:
            got = traffic_gb / avg_launch_s
            hbm = {"achieved": got, "peak": hbm_peak, "unit": "GB/s", "frac": got / hbm_peak,
                   "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    except (OSError, ValueError, KeyError):
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(batch, args.cpu_sample, 1, 0)
        cpu = {"value": cb["value"], "unit": cb["unit"], "cores": cb["cores"], "kind": cb["kind"],
               "sample": cb["sample"], "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "alignments/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": total_ms_max /
            args.steps, "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
            "vs_baseline": None, "dtype": "u32",
            "data": f"synthetic (bitalign simulate --emit-pairs recipe via the bit-exact C++ port, "
                    f"seed {seed}{' + 1000*rank' if world > 1 and args.scaling == 'weak' else ''})",
            "config": {"workload": cfg_desc, "pairs_per_gpu": n, "pairs_total": int(pairs_all),
                       "window": W, "overlap": O, "k": K, "priority": PRIO,
                       "l2": "inputs 2.8 GB per GPU > 126 MB L2; no flush needed",
                       "parallelism": f"pair-sharded x{world}, no collective"},
            "gcups": gcups, "bases_per_s": bases_all * args.steps / (total_ms_max * 1e-3),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gop/s",
                         "frac": achieved / peak if peak > 0 else None,
                         "traffic": traffic_gb, "traffic_unit": "GB of DRAM read+write per launch "
                         "(ncu --set full capture, profiles/ncu_traffic.json)",
                         "ops_per_launch": work.alu_ops,
                         "definition": "5*sum_w (d_min+1)*n_w*ceil(m_w/32) int32 ops per launch "
                                       "/ mean CUDA-event launch time; peak = live LOP3+SHF "
                                       "microbenchmark (ga_bench_alu_peak)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "alignments/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                    "path": "ga_align_batch (C-ABI) on pinned host buffers: 1 byte/symbol in, "
                            "results + distances + 2-bit ops out, chunked copy/kernel overlap",
                    "packed_input": {"value": e2e_pk_value, "h2d_bytes_per_step": h2d_pk,
                                     "path": "same call with ga_batch_in.packed2 (sequences "
                                             "held 2 bits/symbol on the host; packing not timed)"},
                    "host_pack": {"value": e2e_hp_value,
                                  "h2d_bytes_per_step": h2d_pk - 8 * int(packed.exceptions.shape[0]),
                                  "path": "same call on the same byte input with ga_batch_in.packed2 "
                                          "= GA_PACK_HOST (each chunk packed to 2 bits on the host "
                                          "inside the call, timed)"}},
            "gpu_launches": launches, "clocks": clock_info,
            "extra": {"hbm": hbm, "status_counts": status_counts, "windows": work.windows,
                      "dc_entries": work.entries, "tb_steps": work.tb_steps,
                      "step_ms": [round(x, 3) for x in step_ms], "gen_s": round(gen_s, 2)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
