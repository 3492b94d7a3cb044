"""Summarise an ncu report: headline metrics, stall reasons, SASS hot spots.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Occupancy",
            "Warp State Statistics", "Scheduler Statistics", "Memory Workload Analysis",
            "Instruction Statistics", "Launch Statistics")
KEEP = ("Duration", "SM Active Cycles", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy",
        "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Achieved Active Warps Per SM", "Theoretical Active Warps per SM",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp",
        "Executed Instructions", "SM Frequency")


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 40
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    si, mi, ui, vi = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    for r in rows[1:]:
        if r[si] in SECTIONS and r[mi] in KEEP:
            print(f"{r[mi]:45s} {r[vi]} {r[ui]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    if raw:
        hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
        stalls = [(hdr[k], vals[k]) for k in range(len(hdr))
                  if hdr[k].startswith("smsp__pcsamp_warps_issue_stalled_") and
                  not hdr[k].endswith("_not_issued")]
        tot = sum(float(v or 0) for _, v in stalls) or 1
        print("-- stall samples --")
        for k, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:10]:
            print(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} "
                  f"{100 * float(v or 0) / tot:5.1f}%")
        for k in range(len(hdr)):
            if hdr[k] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                          "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
                          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                          "smsp__inst_executed.sum"):
                print(f"{hdr[k]:60s} {vals[k]}")
    sass = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv",
                                            "--print-source", "sass"]))))
    if len(sass) > 2:
        h = sass[1]
        ai, si2, ei = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
        st = h.index("Warp Stall Sampling (All Samples)")
        data = [(r[ai], int(r[ei] or 0), int(r[st] or 0), r[si2]) for r in sass[2:] if len(r) > ei]
        tot = sum(d[1] for d in data) or 1
        tots = sum(d[2] for d in data) or 1
        print(f"-- SASS hot spots (of {tot} warp-instructions) --")
        for a, e, s, src in sorted(data, key=lambda x: -x[2])[:nsass]:
            print(f"{a[-5:]} exec{100 * e / tot:5.2f}% stall{100 * s / tots:5.2f}%  {src[:70]}")


if __name__ == "__main__":
    main()
