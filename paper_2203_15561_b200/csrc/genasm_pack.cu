// genasm_pack.cu -- 2-bit transfer formats for the host-buffer path.
//
// The sequences are 2 bits per symbol on the wire (a 4x smaller H2D than one
// byte per symbol) and are expanded to one byte per symbol in HBM by a
// streaming kernel; symbols outside ACGT travel as a sparse exception list.
// The traceback's ops are packed 4 per byte on the device before the D2H.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/genasm.h"

namespace genasm {

// 2-bit -> one code byte per symbol; thread t expands packed bytes [4t, 4t+4)
__global__ void unpack2_kernel(const uint8_t* __restrict__ packed, int64_t nsym,
                               uint8_t* __restrict__ out) {
    const int64_t nbytes = (nsym + 3) >> 2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t * 4 < nbytes;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b0 = t * 4;
        uint32_t w;
        if (b0 + 4 <= nbytes && ((reinterpret_cast<uintptr_t>(packed) & 3) == 0)) {
            w = *reinterpret_cast<const uint32_t*>(packed + b0);
        } else {
            w = 0;
            for (int k = 0; k < 4 && b0 + k < nbytes; ++k) w |= (uint32_t)packed[b0 + k] << (8 * k);
        }
        // 16 symbols: byte k of the output word holds bits 2k..2k+1 of w
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = w >> (8 * q);
            o[q] = (v & 3u) | ((v >> 2) & 3u) << 8 | ((v >> 4) & 3u) << 16 | ((v >> 6) & 3u) << 24;
        }
        const int64_t s0 = b0 * 4;
        if (s0 + 16 <= nsym && ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
            *reinterpret_cast<uint4*>(out + s0) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
            for (int k = 0; k < 16 && s0 + k < nsym; ++k) out[s0 + k] = (uint8_t)(o[k >> 2] >> (8 * (k & 3)));
        }
    }
}

__global__ void patch_exceptions_kernel(const int64_t* __restrict__ pos, int64_t n, int64_t base,
                                        uint8_t* __restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        out[pos[t] - base] = 4;
}

// ASCII ops -> 2-bit codes, 4 per byte; thread t packs ops [16t, 16t+16)
__global__ void pack_ops_kernel(const uint8_t* __restrict__ ascii, int64_t nops,
                                uint8_t* __restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t * 16 < nops;
         t += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int64_t x = t * 16 + k;
            const uint8_t ch = x < nops ? ascii[x] : '=';
            const uint32_t code = (ch == 'X') + 2u * (ch == 'I') + 3u * (ch == 'D');
            w |= code << (2 * k);
        }
        const int64_t b0 = t * 4;
        const int64_t nb = (nops + 3) >> 2;
        for (int k = 0; k < 4 && b0 + k < nb; ++k) out[b0 + k] = (uint8_t)(w >> (8 * k));
    }
}

static int grid_for(int64_t work, int threads) {
    const int64_t g = (work + threads - 1) / threads;
    return (int)(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

cudaError_t launch_unpack2(const uint8_t* packed, int64_t nsym, uint8_t* out, cudaStream_t st) {
    if (nsym <= 0) return cudaSuccess;
    unpack2_kernel<<<grid_for((nsym + 15) / 16, 256), 256, 0, st>>>(packed, nsym, out);
    return cudaGetLastError();
}

cudaError_t launch_patch(const int64_t* pos, int64_t n, int64_t base, uint8_t* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    patch_exceptions_kernel<<<grid_for(n, 256), 256, 0, st>>>(pos, n, base, out);
    return cudaGetLastError();
}

cudaError_t launch_pack_ops(const uint8_t* ascii, int64_t nops, uint8_t* out, cudaStream_t st) {
    if (nops <= 0) return cudaSuccess;
    pack_ops_kernel<<<grid_for((nops + 15) / 16, 256), 256, 0, st>>>(ascii, nops, out);
    return cudaGetLastError();
}

}  // namespace genasm

namespace genasm {
bool host_has_avx2();                                              // pack_host.cpp
int64_t pack2_avx2(const uint8_t* codes, int64_t nblk, uint8_t* out);  // pack_host.cpp
}  // namespace genasm

extern "C" {

// 8 code bytes -> 2 packed bytes (low 2 bits of each code, symbol order kept)
static inline uint32_t pack8(uint64_t v) {
    uint64_t b = v & 0x0303030303030303ull;
    b = (b | (b >> 6)) & 0x000F000F000F000Full;
    b = (b | (b >> 12)) & 0x000000FF000000FFull;
    return (uint32_t)(b & 0xff) | (uint32_t)((b >> 32) & 0xff) << 8;
}

int64_t ga_pack2(const uint8_t* codes, int64_t n, uint8_t* packed, int64_t* exceptions,
                 int64_t max_exceptions) {
    const int64_t nbytes = (n + 3) / 4;
    const int nth = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::min<int>((int)std::thread::hardware_concurrency(), 32),
                             nbytes / (1 << 16)));
    // per-thread ranges of 64 symbols (16 packed bytes)
    const int64_t chunk = ((nbytes + nth - 1) / nth + 15) / 16 * 16;
    std::vector<int64_t> counts((size_t)nth, 0);
    static const bool avx2 = genasm::host_has_avx2();
    auto work = [&](int w) {
        const int64_t b0 = std::min(nbytes, w * chunk), b1 = std::min(nbytes, b0 + chunk);
        int64_t cnt = 0;
        int64_t b = b0;
        if (avx2) {  // 32 symbols per iteration
            const int64_t nblk = std::max<int64_t>(0, std::min(b1 - b0, n / 4 - b0) / 8);
            cnt += genasm::pack2_avx2(codes + 4 * b0, nblk, packed + b0);
            b += 8 * nblk;
        }
        for (; b + 2 <= b1 && 4 * b + 8 <= n; b += 2) {  // 8 symbols per iteration
            uint64_t v;
            memcpy(&v, codes + 4 * b, 8);
            const uint32_t p = pack8(v);
            packed[b] = (uint8_t)p;
            packed[b + 1] = (uint8_t)(p >> 8);
            if (v & 0xFCFCFCFCFCFCFCFCull)
                for (int k = 0; k < 8; ++k) cnt += codes[4 * b + k] > 3;
        }
        for (; b < b1; ++b) {
            uint8_t v = 0;
            for (int k = 0; k < 4 && 4 * b + k < n; ++k) {
                const uint8_t cd = codes[4 * b + k];
                v |= (uint8_t)((cd & 3u) << (2 * k));
                cnt += cd > 3;
            }
            packed[b] = v;
        }
        counts[(size_t)w] = cnt;
    };
    std::vector<int64_t> first((size_t)nth + 1, 0);
    // second pass: each thread lists its range's code-4 positions at its prefix
    auto list = [&](int w) {
        const int64_t x0 = std::min(n, 4 * w * chunk), x1 = std::min(n, x0 + 4 * chunk);
        int64_t k = first[(size_t)w];
        if (!counts[(size_t)w]) return;
        for (int64_t x = x0; x < x1 && k < max_exceptions; ++x)
            if (codes[x] > 3) exceptions[k++] = x;
    };
    auto run = [&](auto&& fn) {
        if (nth == 1) {
            fn(0);
            return;
        }
        std::vector<std::thread> th;
        for (int w = 0; w < nth; ++w) th.emplace_back(fn, w);
        for (auto& t : th) t.join();
    };
    run(work);
    for (int w = 0; w < nth; ++w) first[(size_t)w + 1] = first[(size_t)w] + counts[(size_t)w];
    const int64_t total = first[(size_t)nth];
    if (exceptions && total && max_exceptions > 0) run(list);
    return total;
}

void ga_unpack_ops(const uint8_t* ops2, int64_t first_op, int64_t n_ops, char* out) {
    static const char kOps[4] = {'=', 'X', 'I', 'D'};
    for (int64_t x = 0; x < n_ops; ++x) {
        const int64_t y = first_op + x;
        out[x] = kOps[(ops2[y >> 2] >> (2 * (y & 3))) & 3];
    }
}

}  // extern "C"
