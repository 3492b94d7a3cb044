// Dev microbenchmark: latency per step of the DC wavefront (DcLane) for one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_15561_b200/csrc \
//      -o tools/ubench_dc tools/ubench_dc.cu
#include <cstdio>

#include "genasm_device.cuh"

using namespace genasm;

template <int G, bool PRED>
__global__ void dc_bench(long long* cyc, unsigned* sink, int passes, int warps_active) {
    constexpr int NW = 2;
    using GE = Geo<NW>;
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31, q = lane & (G - 1);
    const int warp = threadIdx.x >> 5;
    if (warp >= warps_active) return;
    const int group = threadIdx.x / G;
    uint32_t* tab = smem + group * (GE::TAB_W + 2 * GE::WMAX * NW);
    uint32_t* carry = tab + GE::TAB_W;
    uint32_t* pmcol = carry + GE::WMAX * NW;
    for (int i = q; i < GE::WMAX * NW; i += G) pmcol[i] = 0x9e3779b9u * (i + 1);
    __syncwarp();
    long long t0 = clock64();
    unsigned acc = 0;
    for (int p = 0; p < passes; ++p) {
        DcLane<NW, G> L;
        L.init(q, true, 0, 64, 64, 64, 64, false, tab, carry, pmcol, nullptr);
        const int steps = 64 + G - 1;
        for (int s = 0; s < G - 1; ++s) L.template step<true, false>(s);
        if (PRED) {
            for (int s = G - 1; s < 64; ++s) L.template step<true, false>(s);
        } else {
#pragma unroll 4
            for (int s = G - 1; s < 64; ++s) L.template step<false, false>(s);
        }
        for (int s = 64; s < steps; ++s) L.template step<true, false>(s);
        acc += L.v[0];
    }
    long long t1 = clock64();
    sink[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / ((long long)passes * (64 + G - 1));
}

int main() {
    long long* cyc;
    unsigned* sink;
    cudaMallocManaged(&cyc, 64);
    cudaMalloc(&sink, 4096);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(dc_bench<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dc_bench<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dc_bench<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int w : {1, 2, 4, 8}) {
        dc_bench<16, false><<<1, 32 * w, smem>>>(cyc, sink, 200, w);
        cudaDeviceSynchronize();
        printf("G=16 steady-unrolled, %d warps/SM: %lld cycles per step\n", w, cyc[0]);
        dc_bench<16, true><<<1, 32 * w, smem>>>(cyc, sink, 200, w);
        cudaDeviceSynchronize();
        printf("G=16 all-predicated,  %d warps/SM: %lld cycles per step\n", w, cyc[0]);
        dc_bench<8, false><<<1, 32 * w, smem>>>(cyc, sink, 200, w);
        cudaDeviceSynchronize();
        printf("G=8  steady-unrolled, %d warps/SM: %lld cycles per step\n", w, cyc[0]);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
