// microbench.cu -- measured int32 logic/shift peak of the running B200, the
// roofline denominator for the DC recurrence (the ALU rate on
// sm_100 is not published, so it is measured live by bench.py).
//
// Each thread runs 8 independent chains of the same op mix the DC emits per
// 32-bit word (LOP3 + funnel shift), so the issue rate is bounded by the ALU
// pipe, not by dependency latency.  ops = threads x iters x 8 x 2.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__global__ void alu_peak_kernel(uint32_t* sink, int iters, uint32_t seed) {
    uint32_t x[8], y = seed ^ threadIdx.x, z = seed * 2654435761u + blockIdx.x;
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = y + c * 0x9e3779b9u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t r;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(r) : "r"(x[c]), "r"(y), "r"(z));
            asm volatile("shf.l.wrap.b32 %0, %1, %2, 1;" : "=r"(x[c]) : "r"(r), "r"(x[(c + 1) & 7]));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc ^= x[c];
    if (acc == 0x12345678u) sink[0] = acc;
}

}  // namespace

extern "C" {

// Returns measured int32 ALU ops/s (best of `reps`), or a negative CUDA error.
double ga_bench_alu_peak(int device, int reps) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint32_t* sink = nullptr;
    if (cudaMalloc(&sink, 16) != cudaSuccess) return -2.0;
    const int threads = 256, blocks = sms * 8, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    alu_peak_kernel<<<blocks, threads>>>(sink, 64, 1u);  // warm-up
    double best = 0.0;
    for (int r = 0; r < (reps > 0 ? reps : 5); ++r) {
        cudaEventRecord(a);
        alu_peak_kernel<<<blocks, threads>>>(sink, iters, (uint32_t)r + 7u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * iters * 8.0 * 2.0;
        const double rate = ops / (ms * 1e-3);
        if (rate > best) best = rate;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? best : -3.0;
}

}  // extern "C"
