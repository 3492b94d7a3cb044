// Dev microbenchmark: thread-per-window column-major DC (16 levels in registers)
// with band words stored to global memory in a lane-interleaved layout.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_colmajor tools/ubench_colmajor.cu
#include <cstdint>
#include <cstdio>

constexpr int LV = 16, N = 64;

__device__ __forceinline__ void shl(uint32_t lo, uint32_t hi, uint32_t& rlo, uint32_t& rhi) {
    rlo = lo << 1;
    rhi = __funnelshift_l(lo, hi, 1);
}

template <bool STORE>
__global__ void __launch_bounds__(256) colmajor(uint32_t* tables, uint32_t* sink, int windows) {
    __shared__ uint32_t pmtab[8][5][2];  // per warp: 4 symbol masks + miss
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane < 10) pmtab[warp][lane >> 1][lane & 1] = 0x9e3779b9u * (lane + 3) ^ (warp * 77);
    if (lane == 10) { pmtab[warp][4][0] = ~0u; pmtab[warp][4][1] = ~0u; }
    __syncwarp();
    const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
    uint2* tab = reinterpret_cast<uint2*>(tables) + (size_t)gw * (LV * N / 2) * 32;
    uint32_t acc = 0;
    uint32_t seed = 0x1234567u * (lane + 1) + gw;
    for (int win = 0; win < windows; ++win) {
        uint32_t clo[LV], chi[LV];
#pragma unroll
        for (int d = 0; d < LV; ++d) {  // init(m, d): bits < d are 0
            clo[d] = ~((1u << d) - 1u);
            chi[d] = ~0u;
        }
        uint32_t keep_lo[LV];
#pragma unroll 1
        for (int j = 0; j < N; j += 2) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                seed = seed * 1664525u + 1013904223u;
                const int code = (seed >> 28) & 3;
                const uint32_t pml = pmtab[warp][code][0], pmh = pmtab[warp][code][1];
                const int amt = min(max(j + h - 16, 0), 32);
                uint32_t plo = clo[0], phi = chi[0];  // R[d-1][j-1]
                uint32_t slo, shi;
                shl(clo[0], chi[0], slo, shi);
                clo[0] = slo | pml;
                chi[0] = shi | pmh;
                uint32_t blo = clo[0], bhi = chi[0];  // R[d-1][j]
                uint32_t band = __funnelshift_rc(clo[0], chi[0], amt);
                if (h == 0) keep_lo[0] = band;
                else if (STORE) tab[((0 * (N / 2) + (j >> 1)) << 5) + lane] = make_uint2(keep_lo[0], band);
                else acc ^= band + keep_lo[0];
#pragma unroll
                for (int d = 1; d < LV; ++d) {
                    const uint32_t alo = plo, ahi = phi;
                    plo = clo[d];
                    phi = chi[d];
                    uint32_t tlo = alo & blo, thi = ahi & bhi, stlo, sthi, svlo, svhi;
                    shl(tlo, thi, stlo, sthi);
                    shl(clo[d], chi[d], svlo, svhi);
                    clo[d] = (svlo | pml) & (stlo & alo);
                    chi[d] = (svhi | pmh) & (sthi & ahi);
                    blo = clo[d];
                    bhi = chi[d];
                    const uint32_t bd = __funnelshift_rc(clo[d], chi[d], amt);
                    if (h == 0) keep_lo[d] = bd;
                    else if (STORE) tab[((d * (N / 2) + (j >> 1)) << 5) + lane] = make_uint2(keep_lo[d], bd);
                    else acc ^= bd + keep_lo[d];
                }
            }
        }
#pragma unroll
        for (int d = 0; d < LV; ++d) acc += clo[d] ^ chi[d];
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int sms = 148, threads = 256, windows = 200;
    const int blocks = sms;
    uint32_t *tables, *sink;
    const size_t words = (size_t)blocks * (threads / 32) * LV * N * 32;
    cudaMalloc(&tables, words * 4);
    cudaMalloc(&sink, (size_t)blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int store = 0; store < 2; ++store) {
        for (int bpsm : {1, 2}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (store) colmajor<true><<<blocks * bpsm, threads>>>(tables, sink, windows / bpsm);
                else colmajor<false><<<blocks * bpsm, threads>>>(tables, sink, windows / bpsm);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double wins = (double)blocks * threads * windows;
                if (rep)
                    printf("store=%d blocks/SM=%d: %.3f ms, %.1f M windows/s, %.2f ns/window/SM, "
                           "entries %.2f T/s\n",
                           store, bpsm, ms, wins / ms / 1e3, ms * 1e6 / (wins / sms),
                           wins * LV * N / (ms * 1e-3) / 1e12);
            }
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
