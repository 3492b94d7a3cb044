// coop_bench.cu -- dev microbenchmark of the full tier's warp-cooperative DC
// and traceback (coop_dc / coop_tb of genasm_thread.cu) on synthetic W = 64
// windows, with the kernel's own code included verbatim.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2203_15561_b200/csrc -o tools/_coop_bench tools/coop_bench.cu
//   tools/_coop_bench [error_rate] [warps_per_sm] [windows_per_warp] [tb: 1, 0 = DC only]
//   tools/_coop_bench c    (shuffle-chain latency probes)
//
// Prints cycles per window (clock64 around each call, averaged over warps)
// and checks every d_min against the host restatement (thr::dc_full).
#include "genasm_thread.cu"

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using namespace genasm;

namespace {
struct HostFullTab {
    std::vector<uint64_t> rows;  // [level][column]
    int n;
    explicit HostFullTab(int K, int n_) : rows((size_t)(K + 8) * 65, 0), n(n_) {}
    uint64_t get(int d, int j) const { return rows[(size_t)d * 65 + j]; }
    void put4(int d0, int j, const uint32_t* lo, const uint32_t* hi) {
        for (int k = 0; k < 4; ++k) rows[(size_t)(d0 + k) * 65 + j] = (uint64_t)hi[k] << 32 | lo[k];
    }
};
}  // namespace

__global__ void __launch_bounds__(128) coop_bench_kernel(const thr::Planes* pp, const thr::Planes* tp,
                                                         int nwin, int reps, int K, uint64_t* tabs,
                                                         int* dmin_out, unsigned long long* cyc,
                                                         uint64_t prio_lut, uint8_t* ops, int variant) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t* tab = tabs + (size_t)gw * (kBandWordsPerWarp / 2);
    __shared__ uint2 s_pm[4][128];
    uint2* pmt = s_pm[threadIdx.x >> 5];
    unsigned long long tdc = 0, ttb = 0;
    for (int r = 0; r < reps; ++r) {
        const int w = (gw * 7 + r) % nwin;
        const thr::Planes p = pp[w], t = tp[w];
        const long long c0 = clock64();
        const int d = coop_dc(p, t, 64, 64, K, K, tab, pmt, lane);
        const long long c1 = clock64();
        if (d >= 0 && variant != 0) {
            int64_t nops = 0;
            thr::TbOut o;
            coop_tb(tab, p, t, 64, 64, d, 40, prio_lut, ops + (size_t)gw * 256, nops, o, lane);
        }
        const long long c2 = clock64();
        __syncwarp();
        tdc += c1 - c0;
        ttb += c2 - c1;
        if (gw == 0 && lane == 0) dmin_out[w] = d;
    }
    if (lane == 0) {
        atomicAdd(cyc, tdc);
        atomicAdd(cyc + 1, ttb);
    }
}

__global__ void shfl_lat_kernel(unsigned long long* out, int iters) {
    uint32_t v = threadIdx.x, w = threadIdx.x * 3;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        v = __shfl_up_sync(FULL, v, 1);
        w = thr::and3(v, w, 0x7fffffffu) + 1;
        v ^= w;
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) out[0] = (c1 - c0) / iters;
    if (v == 12345) out[1] = w;
}

template <int kMode>
__global__ void chain_kernel(unsigned long long* out, int iters, uint64_t* sink) {
    __shared__ uint2 pm[64];
    const int lane = threadIdx.x & 31;
    pm[lane] = make_uint2(lane * 77, lane * 13);
    pm[lane + 32] = make_uint2(lane * 7, lane * 3);
    __syncwarp();
    uint32_t ol = threadIdx.x, oh = threadIdx.x * 3, cl = 5, ch = 9;
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t bl = __shfl_up_sync(FULL, ol, 1);
        uint32_t bh = kMode >= 1 ? __shfl_up_sync(FULL, oh, 1) : ol;
        uint2 p = kMode >= 2 ? pm[(i + lane) & 63] : make_uint2(i, i);
        const uint32_t nl = thr::and3(thr::orand(cl << 1, p.x, bl << 1), bl, cl);
        const uint32_t nh = thr::and3(thr::orand(ch << 1, p.y, bh << 1), bh, ch);
        cl = nl; ch = nh; ol = nl; oh = nh;
        if (kMode >= 3) sink[(size_t)(i & 127) * 32 + lane] = (uint64_t)nh << 32 | nl;
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) out[kMode] = (c1 - c0) / iters;
    if (ol == 12345) sink[0] = oh;
}

int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'c') {
        unsigned long long* o;
        uint64_t* sink;
        cudaMalloc(&o, 64);
        cudaMalloc(&sink, 128 * 32 * 8);
        chain_kernel<0><<<1, 32>>>(o, 10000, sink);
        chain_kernel<1><<<1, 32>>>(o, 10000, sink);
        chain_kernel<2><<<1, 32>>>(o, 10000, sink);
        chain_kernel<3><<<1, 32>>>(o, 10000, sink);
        cudaDeviceSynchronize();
        unsigned long long h1[4];
        cudaMemcpy(h1, o, 32, cudaMemcpyDeviceToHost);
        printf("1 warp: %llu %llu %llu %llu\n", h1[0], h1[1], h1[2], h1[3]);
        chain_kernel<0><<<1, 128>>>(o, 10000, sink);
        chain_kernel<1><<<1, 128>>>(o, 10000, sink);
        chain_kernel<2><<<1, 128>>>(o, 10000, sink);
        chain_kernel<3><<<1, 128>>>(o, 10000, sink);
        unsigned long long h[4];
        cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
        printf("chain cycles/iter: 1 shfl %llu, 2 shfl %llu, +LDS %llu, +STG %llu\n", h[0], h[1], h[2], h[3]);
        return 0;
    }
    if (argc > 1 && argv[1][0] == 's') {
        unsigned long long* o;
        cudaMalloc(&o, 16);
        shfl_lat_kernel<<<1, 32>>>(o, 10000);
        unsigned long long h[2];
        cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("SHFL.UP + LOP3 + IADD + LOP chain: %llu cycles per iteration\n", h[0]);
        return 0;
    }
    const double err = argc > 1 ? atof(argv[1]) : 0.3;
    const int wps = argc > 2 ? atoi(argv[2]) : 4;
    const int reps = argc > 3 ? atoi(argv[3]) : 200;
    const int variant = argc > 4 ? atoi(argv[4]) : 1;
    const int nwin = 512, K = 64;
    std::mt19937 g(7);
    std::vector<thr::Planes> hp(nwin), ht(nwin);
    std::vector<int> hd(nwin);
    for (int w = 0; w < nwin; ++w) {
        uint8_t p[64], t[64];
        for (int i = 0; i < 64; ++i) p[i] = g() & 3;
        int i = 0, o = 0;
        while (o < 64) {  // substitutions / insertions / deletions at rate err
            const double u = std::uniform_real_distribution<double>(0, 1)(g);
            if (u < err / 3 && i < 64) { t[o++] = (p[i++] + 1 + g() % 3) & 3; }
            else if (u < 2 * err / 3) { t[o++] = g() & 3; }
            else if (u < err) { ++i; }
            else { t[o++] = i < 64 ? p[i++] : g() & 3; }
        }
        hp[w] = thr::load_planes(p, 64);
        ht[w] = thr::load_planes(t, 64);
        HostFullTab tab(K, 64);
        hd[w] = thr::dc_full(hp[w], ht[w], 64, 64, K, tab);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * wps / 4;
    thr::Planes *dp, *dt;
    uint64_t* tabs;
    int* dd;
    unsigned long long* cyc;
    uint8_t* ops;
    cudaMalloc(&dp, nwin * sizeof(thr::Planes));
    cudaMalloc(&dt, nwin * sizeof(thr::Planes));
    cudaMalloc(&tabs, (size_t)blocks * 4 * (kBandWordsPerWarp / 2) * 8);
    cudaMalloc(&dd, nwin * 4);
    cudaMalloc(&cyc, 16);
    cudaMalloc(&ops, (size_t)blocks * 4 * 256);
    cudaMemcpy(dp, hp.data(), nwin * sizeof(thr::Planes), cudaMemcpyHostToDevice);
    cudaMemcpy(dt, ht.data(), nwin * sizeof(thr::Planes), cudaMemcpyHostToDevice);
    cudaMemset(dd, 0xff, nwin * 4);
    cudaMemset(cyc, 0, 16);
    // MSID priority LUT: okm -> first of M, S, I, D present
    uint64_t lut = 0;
    for (int m = 0; m < 16; ++m) {
        int op = 5;
        for (int e = 0; e < 4; ++e)
            if (m >> e & 1) { op = e; break; }
        lut |= (uint64_t)op << (4 * m);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    coop_bench_kernel<<<blocks, 128>>>(dp, dt, nwin, reps, K, tabs, dd, cyc, lut, ops, variant);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<int> gd(nwin);
    unsigned long long hc[2];
    cudaMemcpy(gd.data(), dd, nwin * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
    int bad = 0, seen = 0;
    double dsum = 0;
    for (int w = 0; w < nwin; ++w) {
        if (gd[w] == -2 + 1 && false) continue;
        if (gd[w] != -1 || hd[w] == -1) {
            if (gd[w] != (int)0xffffffff) ++seen;
        }
        if (gd[w] != hd[w] && gd[w] != -1) ++bad;
        dsum += hd[w];
    }
    const double wins = (double)blocks * 4 * reps;
    printf("v%d err %.2f warps/SM %d: %s, mean d_min %.1f, mismatches %d/%d; DC %.0f TB %.0f cycles/window, "
           "%.3f ms, %.2f M windows/s\n",
           variant, err, wps, cudaGetErrorString(e), dsum / nwin, bad, seen, hc[0] / wins, hc[1] / wins, ms,
           wins / ms / 1e3);
    return bad != 0;
}
