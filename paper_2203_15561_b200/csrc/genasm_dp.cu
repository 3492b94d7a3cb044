// genasm_dp.cu -- the ground-truth distances of the `bench` accuracy columns
// on the device: oracle.global_distance / semiglobal_distance
// (pkg/src/bitalign/oracle.py:24-74; the classical quadratic DP with
// dp[i][0] = i and dp[0][j] = j, or 0 with a free text prefix).
//
// Bit-vector formulation of the same DP (Myers 1999 / Hyyro 2003): per text
// column, the vertical deltas of 64 rows at a time (VP/VN words), the
// horizontal delta carried from block to block, the bottom row's score
// updated by the last block's delta at row m-1.  Equal symbol ids match
// (characters, not the aligner's codes: 'N' matches 'N' here as in the
// reference's DP).  One lane per pair, pairs from an atomic queue; the VP/VN
// and match-mask words live in a per-lane global slab interleaved across
// lanes ([word][lane]) so a warp's accesses coalesce.
#include "genasm_kernel.cuh"

namespace genasm {

namespace {

constexpr int kDBlock = 128;

// one 64-row block of one column; returns the horizontal delta out of its
// row `top` (63, or (m-1)&63 in the last block)
__device__ __forceinline__ int dp_block(uint64_t& vp, uint64_t& vn, uint64_t eq, int hin, int top) {
    const uint64_t neg = hin < 0 ? 1ull : 0ull;
    const uint64_t xv = eq | vn;
    eq |= neg;
    const uint64_t xh = (((eq & vp) + vp) ^ vp) | eq;
    uint64_t ph = vn | ~(xh | vp);
    uint64_t mh = vp & xh;
    const int hout = (int)((ph >> top) & 1ull) - (int)((mh >> top) & 1ull);
    ph = (ph << 1) | (hin > 0 ? 1ull : 0ull);
    mh = (mh << 1) | neg;
    vp = mh | ~(xv | ph);
    vn = ph & xv;
    return hout;
}

__global__ void __launch_bounds__(kDBlock)
edit_distance_kernel(const uint8_t* syms, const int64_t* pat_off, const int32_t* pat_len,
                     const int64_t* txt_off, const int32_t* txt_len, const int32_t* order,
                     int64_t n_pairs, int semiglobal, int64_t* dist, uint64_t* slab, int64_t lanes,
                     unsigned long long* queue) {
    const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    for (;;) {
        const unsigned long long qi = atomicAdd(queue, 1ull);
        if (qi >= (unsigned long long)n_pairs) break;
        const int q = order ? order[qi] : (int)qi;
        const int m = pat_len[q], n = txt_len[q];
        if (m <= 0) {
            dist[q] = semiglobal ? -1 : n;  // semiglobal_distance raises on an empty pattern
            continue;
        }
        const uint8_t* P = syms + pat_off[q];
        const uint8_t* T = syms + txt_off[q];
        const int nb = (m + 63) >> 6;
        // slab words of this lane: vp[nb] | vn[nb] | peq[4][nb], each [word][lane]
        auto at = [&](int64_t w) -> uint64_t& { return slab[w * lanes + lane]; };
        for (int b = 0; b < nb; ++b) {
            uint64_t e[4] = {0, 0, 0, 0};
            const int hi = m - 64 * b < 64 ? m - 64 * b : 64;
            for (int i = 0; i < hi; ++i) {
                const uint8_t s = P[64 * b + i];
                if (s < 4) e[s] |= 1ull << i;
            }
            at(b) = ~0ull;
            at(nb + b) = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) at((2 + c) * (int64_t)nb + b) = e[c];
        }
        const int last = (m - 1) & 63;
        int64_t score = m;
        for (int j = 0; j < n; ++j) {
            const uint8_t c = T[j];
            int h = semiglobal ? 0 : 1;
            for (int b = 0; b < nb; ++b) {
                uint64_t eq;
                if (c < 4) {
                    eq = at((2 + c) * (int64_t)nb + b);
                } else {  // any other character: matches only itself
                    eq = 0;
                    const int hi = m - 64 * b < 64 ? m - 64 * b : 64;
                    for (int i = 0; i < hi; ++i) eq |= (uint64_t)(P[64 * b + i] == c) << i;
                }
                uint64_t vp = at(b), vn = at(nb + b);
                h = dp_block(vp, vn, eq, h, b == nb - 1 ? last : 63);
                at(b) = vp;
                at(nb + b) = vn;
            }
            score += h;
        }
        dist[q] = score;
    }
}

}  // namespace

cudaError_t launch_edit_distance(const uint8_t* syms, const int64_t* pat_off, const int32_t* pat_len,
                                 const int64_t* txt_off, const int32_t* txt_len, const int32_t* order,
                                 int64_t n_pairs, int max_words, int semiglobal, int64_t* dist,
                                 int num_sms, cudaStream_t stream, uint64_t** slab, size_t* cap,
                                 unsigned long long* queue) {
    if (n_pairs <= 0) return cudaSuccess;
    // lanes: enough to fill the GPU, bounded so the slab stays within 4 GB
    int64_t lanes = (int64_t)num_sms * 1024;
    if (lanes > n_pairs) lanes = n_pairs;
    const int64_t per_lane = 6ll * (max_words > 0 ? max_words : 1);
    const int64_t max_lanes = (4ll << 30) / 8 / per_lane;
    if (lanes > max_lanes) lanes = max_lanes > 32 ? max_lanes : 32;
    const size_t need = (size_t)(lanes * per_lane);
    cudaError_t e;
    if (need > *cap || !*slab) {
        if (*slab) cudaFree(*slab);
        *slab = nullptr;
        *cap = 0;
        if ((e = cudaMalloc(slab, need * 8))) return e;
        *cap = need;
    }
    if ((e = cudaMemsetAsync(queue, 0, sizeof(unsigned long long), stream))) return e;
    const int grid = (int)((lanes + kDBlock - 1) / kDBlock);
    edit_distance_kernel<<<grid, kDBlock, 0, stream>>>(syms, pat_off, pat_len, txt_off, txt_len, order,
                                                       n_pairs, semiglobal, dist, *slab, lanes, queue);
    return cudaGetLastError();
}

}  // namespace genasm
