// Dev microbenchmark: dependent-chain latencies on the running GPU (1 warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_lat tools/ubench_lat.cu
#include <cstdio>
#include <cstdint>

__global__ void lat(unsigned* out, long long* cyc, unsigned seed) {
    __shared__ unsigned sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i + 1) & 1023;
    __syncwarp();
    unsigned x = seed + threadIdx.x;
    const int N = 4096;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_up_sync(0xffffffffu, x, 1, 16) + 1;
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(seed), "r"(i));
    long long t2 = clock64();
    unsigned p = x & 1023;
    for (int i = 0; i < N; ++i) p = sm[p];
    long long t3 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) ^ i;
    long long t4 = clock64();
    for (int i = 0; i < N; ++i) { asm volatile("shf.l.wrap.b32 %0, %0, %0, 1;" : "+r"(x)); }
    long long t5 = clock64();
    out[threadIdx.x] = x + p;
    if (threadIdx.x == 0) {
        cyc[0] = (t1 - t0) / N;
        cyc[1] = (t2 - t1) / N;
        cyc[2] = (t3 - t2) / N;
        cyc[3] = (t4 - t3) / N;
        cyc[4] = (t5 - t4) / N;
    }
}

int main() {
    unsigned* out;
    long long* cyc;
    cudaMalloc(&out, 128);
    cudaMallocManaged(&cyc, 64);
    lat<<<1, 32>>>(out, cyc, 7);
    lat<<<1, 32>>>(out, cyc, 9);
    cudaDeviceSynchronize();
    printf("cycles per dependent op: shfl.up+add %lld  lop3 %lld  lds %lld  shfl.xor+xor %lld  shf %lld\n",
           cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
    return 0;
}
