#!/bin/sh
# dev build of the extension with the lane-per-pair kernel's counters
# (-DGA_THREAD_STATS) into tools/_genasm_stats.so; use with GA_SO=...
cd "$(dirname "$0")/../paper_2203_15561_b200/csrc" && \
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DGA_THREAD_STATS \
  -Xcompiler -fPIC,-O3,-pthread -shared -cudart static -o ../../tools/_genasm_stats.so \
  genasm_lockstep.cu genasm_thread.cu genasm_capi.cu genasm_pack.cu sim.cpp accounting.cpp microbench.cu genasm_io.cpp genasm_baseline.cu genasm_dp.cu pack_host.cpp
