#!/bin/sh
# dev build of the extension with extra nvcc flags into tools/_genasm_<name>.so
#   tools/build_variant.sh <name> [nvcc flags...]; use with GA_SO=tools/_genasm_<name>.so
name=$1; shift
cd "$(dirname "$0")/../paper_2203_15561_b200/csrc" && \
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 "$@" \
  -Xcompiler -fPIC,-O3,-pthread -shared -cudart static -o ../../tools/_genasm_$name.so \
  genasm_lockstep.cu genasm_thread.cu genasm_capi.cu genasm_pack.cu sim.cpp accounting.cpp microbench.cu genasm_io.cpp genasm_baseline.cu genasm_dp.cu pack_host.cpp
