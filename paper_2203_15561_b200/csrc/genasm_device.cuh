// genasm_device.cuh -- device building blocks shared by the kernels:
// bit-row helpers, the shared-memory geometry, one DC wavefront lane, group
// reductions.  See genasm_kernel.cuh for the design.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "genasm_kernel.cuh"

namespace genasm {

constexpr int kMaxBlock = 256;

enum : int { NEED_PAIR = 0, NEED_WINDOW = 1, IN_DC = 2, IN_TB = 3, DONE = 4 };
enum : int { OP_M = 0, OP_S = 1, OP_I = 2, OP_D = 3, OP_STOP = 4, OP_STUCK = 5 };

// ---- bit rows: NW little-endian 32-bit words, 0 = active ----

// init(m, d): bits < min(d, m) are 0 (bitvec.py:108-122); bits >= m are
// don't-care and left 1.
template <int NW>
__device__ __forceinline__ void init_row(uint32_t (&r)[NW], int m, int d) {
    const int z = d < m ? d : m;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const int lo = 32 * w;
        uint32_t zero;
        if (z >= lo + 32) zero = 0xffffffffu;
        else if (z <= lo) zero = 0u;
        else zero = (1u << (z - lo)) - 1u;
        r[w] = ~zero;
    }
}

// shift toward higher bit index by one, shifting in an active 0 (bitvec.py:68-74)
template <int NW>
__device__ __forceinline__ void shl1(const uint32_t (&x)[NW], uint32_t (&r)[NW]) {
    r[0] = x[0] << 1;
#pragma unroll
    for (int w = 1; w < NW; ++w) r[w] = __funnelshift_l(x[w - 1], x[w], 1);
}

template <int NW>
__device__ __forceinline__ uint32_t word_sel(const uint32_t (&x)[NW], int w) {
    uint32_t v = x[0];
#pragma unroll
    for (int u = 1; u < NW; ++u) v = (w == u) ? x[u] : v;
    return v;
}

// 32-bit band of a row starting at bit `amt` (0 <= amt <= 32*NW-32)
template <int NW>
__device__ __forceinline__ uint32_t band32(const uint32_t (&r)[NW], int amt) {
    if (NW == 1) return r[0];
    if (NW == 2) return __funnelshift_rc(r[0], r[NW - 1], (unsigned)amt);
    const int wi = amt >> 5;
    const int wj = wi + 1 < NW ? wi + 1 : NW - 1;
    return __funnelshift_r(word_sel<NW>(r, wi), word_sel<NW>(r, wj), (unsigned)(amt & 31));
}

template <int NW>
struct Geo {
    static constexpr int WMAX = 32 * NW;
    static constexpr bool BAND = NW >= 2;     // 32-bit band entries (else full 32-bit rows)
    static constexpr int LV = BAND ? 16 : 40;  // table levels resident in shared memory
    static constexpr int TAB_W = LV * WMAX;    // words
    static constexpr int GROUP_W = TAB_W + 2 * WMAX * NW + WMAX / 2;
    static constexpr int BAND_MAX = 32 * NW - 32;
};

constexpr unsigned FULL = 0xffffffffu;

// reductions over the G lanes of a group, all 32 lanes participating
template <int G>
__device__ __forceinline__ unsigned group_sum(unsigned x) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o, G);
    return x;
}
template <int G>
__device__ __forceinline__ unsigned group_or(unsigned x) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) x |= __shfl_xor_sync(FULL, x, o, G);
    return x;
}

// One lane of a multi-level DC wavefront: a group of G lanes covers G*LPL
// consecutive levels per pass; lane q owns levels dq .. dq+LPL-1 with
// dq = pass*G*LPL + q*LPL and at step s evaluates column j = s-q+1 of all of
// them, column-major inside the lane (distance.py:125-149):
//   R[d][j] = (sh(R[d][j-1]) | PM[T[j-1]]) & sh(R[d-1][j-1] & R[d-1][j]) & R[d-1][j-1]
// Level dq takes R[dq-1][j] from lane q-1 by one shuffle (lane 0: the carry
// row of the previous pass); levels dq+1.. use the lane's own registers.  One
// shuffle, one mask load and a few address updates are shared by LPL entries.
// PRED: fill/drain steps where some lanes are outside [1, n]; MIXED: some
// group of the warp stores full-width rows (full mode) this round.
template <int NW, int G, int LPL>
struct DcLaneM {
    using GE = Geo<NW>;
    uint32_t col[LPL][NW], a0[NW], outv[NW], npm[NW], ncw[NW];
    uint32_t lvl0;
    int q, n, dq, K, amt_base;
    bool active, lane0carry, lastlane, full;
    uint32_t* bptr;
    uint32_t* grow;
    uint32_t* crow;
    const uint32_t* prow;

    // the band table lives in global memory, one region per warp, laid out
    // [pass][step][lane][LPL]: at each step the 32 lanes store 32*LPL
    // consecutive words (entry (d, c) of lane q was written at step c + q)
    static constexpr int SMAX = GE::WMAX + G - 1;  // steps per pass
    __device__ __forceinline__ void init(int q_, bool in_dc, int pass, int m, int n_, int K_, int W,
                                         bool full_, uint32_t* gband, int lane, uint32_t* carry,
                                         const uint32_t* pmcol, uint32_t* gtab) {
        q = q_;
        n = n_;
        K = K_;
        dq = pass * G * LPL + q * LPL;
        bptr = gband + ((int64_t)pass * SMAX * 32 + lane) * LPL;
        active = in_dc && dq <= K;
        lane0carry = active && q == 0 && dq > 0;
        lastlane = active && q == G - 1;
        full = full_;
#pragma unroll
        for (int k = 0; k < LPL; ++k) init_row<NW>(col[k], m, dq + k);  // R[d][0] = init(m, d)
        init_row<NW>(a0, m, dq > 0 ? dq - 1 : 0);                          // R[dq-1][0]
        lvl0 = dq == 0 ? 0xffffffffu : 0u;  // level 0 has only the match edge
#pragma unroll
        for (int w = 0; w < NW; ++w) outv[w] = 0u;
        amt_base = m - n - 15 - q;  // band origin of column j = s-q+1
        grow = gtab + (int64_t)dq * W * NW;
        gstride_ = (int64_t)W * NW;
        crow = carry;
        prow = pmcol;
        // column index c = s - q of step 0; every c in [-(G-1), n+G-1] addresses
        // words inside this group's shared region, so the loads need no guard
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            npm[w] = prow[-q * NW + w];
            ncw[w] = crow[-q * NW + w];
        }
    }

    template <bool PRED, bool MIXED>
    __device__ __forceinline__ void step(int s) {
        uint32_t b[NW], pm[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) b[w] = __shfl_up_sync(0xffffffffu, outv[w], 1, G);
        const int c = s - q;  // column j-1
        const bool inr = PRED ? (active && (unsigned)c < (unsigned)n) : active;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            b[w] = lane0carry ? ncw[w] : b[w];
            pm[w] = npm[w];
            npm[w] = prow[(c + 1) * NW + w];  // prefetch the next step's words
            ncw[w] = crow[(c + 1) * NW + w];
        }
        uint32_t nc[LPL][NW];
        {
            uint32_t tt[NW], st[NW], sv[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) tt[w] = a0[w] & b[w];
            shl1<NW>(tt, st);
            shl1<NW>(col[0], sv);
#pragma unroll
            for (int w = 0; w < NW; ++w) nc[0][w] = (sv[w] | pm[w]) & ((st[w] & a0[w]) | lvl0);
        }
#pragma unroll
        for (int k = 1; k < LPL; ++k) {
            uint32_t tt[NW], st[NW], sv[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) tt[w] = col[k - 1][w] & nc[k - 1][w];
            shl1<NW>(tt, st);
            shl1<NW>(col[k], sv);
#pragma unroll
            for (int w = 0; w < NW; ++w) nc[k][w] = (sv[w] | pm[w]) & st[w] & col[k - 1][w];
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            a0[w] = PRED ? (inr ? b[w] : a0[w]) : b[w];
            outv[w] = PRED ? (inr ? nc[LPL - 1][w] : outv[w]) : nc[LPL - 1][w];
        }
#pragma unroll
        for (int k = 0; k < LPL; ++k)
#pragma unroll
            for (int w = 0; w < NW; ++w) col[k][w] = PRED ? (inr ? nc[k][w] : col[k][w]) : nc[k][w];
        if (inr && !(MIXED && full)) {
            int amt = amt_base + s;
            amt = amt < 0 ? 0 : amt;
            if (NW > 2) amt = amt > GE::BAND_MAX ? GE::BAND_MAX : amt;
            uint32_t bw[LPL];
#pragma unroll
            for (int k = 0; k < LPL; ++k) bw[k] = GE::BAND ? band32<NW>(nc[k], amt) : nc[k][0];
            uint32_t* dst = bptr + (int64_t)s * 32 * LPL;
            if (LPL == 4) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(bw[0], bw[LPL > 1 ? 1 : 0],
                                                            bw[LPL > 2 ? 2 : 0], bw[LPL > 3 ? 3 : 0]);
            } else if (LPL == 2) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(bw[0], bw[LPL > 1 ? 1 : 0]);
            } else {
#pragma unroll
                for (int k = 0; k < LPL; ++k) dst[k] = bw[k];
            }
        }
        if (MIXED && full && inr) {
#pragma unroll
            for (int k = 0; k < LPL; ++k)
#pragma unroll
                for (int w = 0; w < NW; ++w) grow[gstride_ * k + c * NW + w] = nc[k][w];
        }
        if (lastlane && inr) {
#pragma unroll
            for (int w = 0; w < NW; ++w) crow[c * NW + w] = nc[LPL - 1][w];
        }
    }

    // lowest level of this lane whose column-n row has bit m-1 clear (or -1)
    __device__ __forceinline__ int first_success(int m) const {
        if (!active || n < 1) return -1;
        const int tw = (m - 1) >> 5;
        const uint32_t tb = 1u << ((m - 1) & 31);
        int f = -1;
#pragma unroll
        for (int k = LPL - 1; k >= 0; --k)
            if ((word_sel<NW>(col[k], tw) & tb) == 0u && dq + k <= K) f = k;
        return f;
    }

    int64_t gstride_ = 0;  // words between consecutive levels in the full-mode slab
};

}  // namespace genasm
