// genasm_kernel.cu -- fused windowed GenASM-DC + GenASM-TB kernel (sm_100a).
// See genasm_kernel.cuh for the design summary and DESIGN.md for the roofline.
#include <cuda_runtime.h>
#include <stdint.h>

#include "genasm_kernel.cuh"

namespace genasm {

constexpr int kBlockThreads = 128;

// ---- bit-row helpers (rows are NW little-endian 32-bit words, 0 = active) ----

// init(m, d): bits < min(d, m) are 0 (bitvec.py:108-122).  Bits >= m are
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

__device__ __forceinline__ uint32_t bit_of(const uint32_t* e, int x) {
    return (e[x >> 5] >> (x & 31)) & 1u;
}

template <int NW, int G>
__global__ void __launch_bounds__(kBlockThreads)
genasm_window_kernel(const KernelParams P) {
    extern __shared__ uint32_t smem[];
    constexpr int WMAX = 32 * NW;
    const int lane = threadIdx.x & 31;
    const int q = lane & (G - 1);
    const int gbase = lane & ~(G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
    const unsigned lowmask = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
    const int groups_per_block = kBlockThreads / G;
    const int group_in_block = threadIdx.x / G;
    const int W = P.W, O = P.O, K = P.k, S = P.s_lv;

    const int tab_words = S * W * NW;
    const int group_words = tab_words + WMAX * NW + WMAX / 2;
    uint32_t* tab = smem + group_in_block * group_words;
    uint32_t* pmcol = tab + tab_words;
    uint8_t* cp = reinterpret_cast<uint8_t*>(pmcol + WMAX * NW);
    uint8_t* ct = cp + WMAX;
    const int64_t gid = (int64_t)blockIdx.x * groups_per_block + group_in_block;
    uint32_t* gtab = P.overflow + gid * P.overflow_words_per_group;

    auto entry = [&](int d, int j) -> uint32_t* {  // j in 1..n
        return d < S ? tab + (d * W + (j - 1)) * NW : gtab + ((d - S) * W + (j - 1)) * NW;
    };

    PairResult* results = reinterpret_cast<PairResult*>(P.results);

    for (;;) {
        unsigned long long idx = 0;
        if (q == 0) idx = atomicAdd(P.queue, 1ull);
        idx = __shfl_sync(gmask, idx, 0, G);
        if (idx >= (unsigned long long)P.n_pairs) break;
        const int64_t pair = P.order ? (int64_t)P.order[idx] : (int64_t)idx;
        const int32_t Lp = P.pat_len[pair];
        const int32_t Lt = P.txt_len[pair];
        const uint8_t* Pp = P.codes + P.pat_off[pair];
        const uint8_t* Tp = P.codes + P.txt_off[pair];
        uint8_t* ops = P.ops + P.ops_off[pair];
        uint8_t* dists = P.dists + P.win_off[pair];

        PairResult res;
        res.status = 0; res.fail_window = -1; res.cost = 0; res.text_consumed = 0;
        res.rows_computed = 0; res.ops_len = 0; res.entry_reads = 0; res.entry_writes = 0;
        res.words_allocated = 0;
        if (Lp <= 0) {
            res.status = 2;  // EmptyPattern (window.py:87-88)
            if (q == 0) results[pair] = res;
            continue;
        }

        int64_t p = 0, t = 0;
        int widx = 0;
        while (p < Lp) {
            // ---- window geometry (window.py:96-101) ----
            const int64_t remaining = Lp - p;
            const bool final_w = remaining <= W;
            const int m = final_w ? (int)remaining : W;
            const int64_t tleft = Lt - t;
            const int n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
            const int budget = final_w ? m : W - O;

            // ---- stage reversed chunks (window.py:99-100) ----
            __syncwarp(gmask);
            for (int i = q; i < m; i += G) cp[i] = Pp[p + m - 1 - i];
            for (int j = q; j < n; j += G) ct[j] = Tp[t + n - 1 - j];
            __syncwarp(gmask);

            // ---- pattern masks (distance.py:70-79) and per-column masks (:91-94) ----
            uint32_t mt[4][NW];
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int w = 0; w < NW; ++w) mt[c][w] = 0u;
            for (int i = q; i < m; i += G) {
                const int c = cp[i];
                const uint32_t bit = 1u << (i & 31);
                const int wi = i >> 5;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                    for (int w = 0; w < NW; ++w) mt[cc][w] |= (c == cc && wi == w) ? bit : 0u;
            }
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                for (int w = 0; w < NW; ++w) mt[cc][w] = ~__reduce_or_sync(gmask, mt[cc][w]);
            for (int j = q; j < n; j += G) {
                const int c = ct[j];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    uint32_t x = 0xffffffffu;
                    x = (c == 0) ? mt[0][w] : x;
                    x = (c == 1) ? mt[1][w] : x;
                    x = (c == 2) ? mt[2][w] : x;
                    x = (c == 3) ? mt[3][w] : x;
                    pmcol[j * NW + w] = x;
                }
            }
            __syncwarp(gmask);

            // ---- GenASM-DC: levels-as-lanes wavefront with early termination ----
            int d_min = -1;
            if (n == 0) {
                d_min = m <= K ? m : -1;  // R[d][0] = init(m,d) solves iff d >= m
            } else {
                const int topw = (m - 1) >> 5;
                const uint32_t topb = 1u << ((m - 1) & 31);
                for (int pass = 0; pass * G <= K; ++pass) {
                    const int d = pass * G + q;
                    const bool active = d <= K;
                    uint32_t v[NW], a[NW], outv[NW];
                    init_row<NW>(v, m, d);
                    init_row<NW>(a, m, d - 1 < 0 ? 0 : d - 1);
#pragma unroll
                    for (int w = 0; w < NW; ++w) outv[w] = 0u;
                    bool succ = false;
                    const int steps = n + G - 1;
                    for (int s = 0; s < steps; ++s) {
                        const int j = s - q + 1;
                        uint32_t b[NW];
#pragma unroll
                        for (int w = 0; w < NW; ++w) b[w] = __shfl_up_sync(gmask, outv[w], 1, G);
                        const bool inrange = active && j >= 1 && j <= n;
                        if (inrange) {
                            if (q == 0 && d >= 1) {
                                const uint32_t* src = entry(d - 1, j);
#pragma unroll
                                for (int w = 0; w < NW; ++w) b[w] = src[w];
                            }
                            uint32_t sv[NW], r[NW];
                            shl1<NW>(v, sv);
                            const uint32_t* pm = pmcol + (j - 1) * NW;
                            if (d == 0) {
#pragma unroll
                                for (int w = 0; w < NW; ++w) r[w] = sv[w] | pm[w];
                            } else {
                                uint32_t tt[NW], st[NW];
#pragma unroll
                                for (int w = 0; w < NW; ++w) tt[w] = a[w] & b[w];
                                shl1<NW>(tt, st);
#pragma unroll
                                for (int w = 0; w < NW; ++w) {
                                    r[w] = (sv[w] | pm[w]) & st[w] & a[w];
                                    a[w] = b[w];
                                }
                            }
                            uint32_t* dst = entry(d, j);
#pragma unroll
                            for (int w = 0; w < NW; ++w) {
                                dst[w] = r[w];
                                v[w] = r[w];
                                outv[w] = r[w];
                            }
                            if (j == n) succ = (word_sel<NW>(r, topw) & topb) == 0u;
                        }
                    }
                    const unsigned bal = (__ballot_sync(gmask, succ) >> gbase) & lowmask;
                    // the overflow writes of this pass must be visible to lane 0 of the next
                    __syncwarp(gmask);
                    if (bal) {
                        d_min = pass * G + __ffs(bal) - 1;
                        break;
                    }
                }
            }
            if (d_min < 0) {  // NotFound(k) -> WindowFailed(index, k) (window.py:108-109)
                res.status = 1;
                res.fail_window = widx;
                break;
            }

            // ---- GenASM-TB (backtrace.py:113-160), lane 0 walks ----
            int consumed = 0, tcons = 0, stuck = 0;
            if (q == 0) {
                int j = n, d = d_min, i = m - 1;
                int64_t nops = res.ops_len;
                for (;;) {
                    if (i < 0) break;
                    if (consumed >= budget) break;
                    if (j == 0) {
                        if (i + 1 > d) { stuck = 1; break; }
                        const int take = (i + 1 < budget - consumed) ? i + 1 : budget - consumed;
                        for (int u = 0; u < take; ++u) ops[nops++] = 'I';
                        res.cost += take;
                        consumed += take;
                        i -= take;
                        break;
                    }
                    const int tc = ct[j - 1];
                    const bool sym_eq = tc < 4 && cp[i] == tc;
                    bool m_ok;
                    if (i == 0) m_ok = sym_eq;
                    else if (j == 1) m_ok = sym_eq && (i - 1 < d);
                    else m_ok = sym_eq && !bit_of(entry(d, j - 1), i - 1);
                    res.entry_reads += (j - 1 >= 1);
                    bool s_ok = false, d_ok = false, i_ok = false;
                    if (d > 0) {
                        if (j == 1) {
                            s_ok = (i == 0) || (i - 1 < d - 1);
                            d_ok = i < d - 1;
                        } else {
                            const uint32_t* e = entry(d - 1, j - 1);
                            s_ok = (i == 0) || !bit_of(e, i - 1);
                            d_ok = !bit_of(e, i);
                            res.entry_reads += 1;
                        }
                        i_ok = (i == 0) || !bit_of(entry(d - 1, j), i - 1);
                        res.entry_reads += 1;
                    }
                    int op = -1;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int id = (P.prio >> (2 * u)) & 3;
                        const bool ok = id == 0 ? m_ok : id == 1 ? s_ok : id == 2 ? i_ok : d_ok;
                        if (op < 0 && ok) op = id;
                    }
                    if (op == 0) {
                        ops[nops++] = '='; --j; --i; ++consumed; ++tcons;
                    } else if (op == 1) {
                        ops[nops++] = 'X'; --j; --d; --i; ++consumed; ++tcons; ++res.cost;
                    } else if (op == 2) {
                        ops[nops++] = 'I'; --d; --i; ++consumed; ++res.cost;
                    } else if (op == 3) {
                        ops[nops++] = 'D'; --j; --d; ++tcons; ++res.cost;
                    } else {
                        stuck = 1;
                        break;
                    }
                }
                res.ops_len = nops;
                dists[widx] = (uint8_t)d_min;
                res.rows_computed += d_min + 1;
                // entry_writes / words_allocated in closed form
                int64_t wr = 0;
                for (int dd = 0; dd <= d_min; ++dd) {
                    int ss = n - budget - (K - dd) - 1;
                    ss = ss > 1 ? ss : 1;
                    const int cnt = n - ss + 1;
                    wr += cnt > 0 ? cnt : 0;
                }
                res.entry_writes += wr;
                res.words_allocated += wr * ((m + 63) / 64);
            }
            consumed = __shfl_sync(gmask, consumed, 0, G);
            tcons = __shfl_sync(gmask, tcons, 0, G);
            stuck = __shfl_sync(gmask, stuck, 0, G);
            if (stuck) {
                res.status = 3;
                res.fail_window = widx;
                break;
            }
            p += consumed;
            t += tcons;
            ++widx;
        }
        if (q == 0) {
            res.text_consumed = t;
            if (res.status != 0) {  // a failed slot carries only its error (window.py:144-149)
                const int32_t st = res.status, fw = res.fail_window;
                res = PairResult{};
                res.status = st;
                res.fail_window = fw;
            }
            results[pair] = res;
        }
    }
}

// ---------------------------------------------------------------------------

template <int NW, int G>
static cudaError_t launch_t(const KernelParams& base, int s_lv, int smem_budget, int num_sms,
                            cudaStream_t stream,
                            uint32_t** overflow, size_t* overflow_cap, LaunchShape* shape) {
    constexpr int WMAX = 32 * NW;
    KernelParams P = base;
    const int groups_per_block = kBlockThreads / G;
    // shared-memory table depth: requested levels, capped so one block fits
    // in the per-block budget (GA_SMEM_KB) -- deeper levels use the overflow
    const int levels_cap = ((P.k + 1 + G - 1) / G) * G;
    const int fixed_words = WMAX * NW + WMAX / 2;
    const int level_words = P.W * NW;
    const int fit = (smem_budget / 4 / groups_per_block - fixed_words) / level_words;
    if (s_lv > fit) s_lv = fit;
    if (s_lv > levels_cap) s_lv = levels_cap;
    if (s_lv < 0) s_lv = 0;
    P.s_lv = s_lv;
    const int group_words = s_lv * P.W * NW + WMAX * NW + WMAX / 2;
    const int smem = groups_per_block * group_words * 4;
    auto kern = genasm_window_kernel<NW, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlockThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t groups_needed = (P.n_pairs + 0);
    int grid = num_sms * per_sm;
    const int64_t max_useful = (groups_needed + groups_per_block - 1) / groups_per_block;
    if (grid > max_useful) grid = (int)(max_useful > 0 ? max_useful : 1);
    const int64_t ovf_levels = levels_cap > s_lv ? levels_cap - s_lv : 0;
    P.overflow_words_per_group = ovf_levels * P.W * NW;
    const size_t need = (size_t)grid * groups_per_block * (size_t)P.overflow_words_per_group;
    if (need > *overflow_cap) {
        if (*overflow) cudaFree(*overflow);
        *overflow = nullptr;
        *overflow_cap = 0;
        e = cudaMalloc(overflow, need * 4 + 16);
        if (e != cudaSuccess) return e;
        *overflow_cap = need;
    }
    P.overflow = *overflow;
    kern<<<grid, kBlockThreads, smem, stream>>>(P);
    shape->grid = grid;
    shape->block = kBlockThreads;
    shape->smem_bytes = smem;
    shape->s_lv = s_lv;
    shape->group = G;
    shape->overflow_words_per_group = P.overflow_words_per_group;
    return cudaGetLastError();
}

template <int NW>
static cudaError_t launch_nw(const KernelParams& P, int group, int s_lv, int sb, int num_sms,
                             cudaStream_t stream, uint32_t** overflow, size_t* cap,
                             LaunchShape* shape) {
    switch (group) {
        case 8: return launch_t<NW, 8>(P, s_lv, sb, num_sms, stream, overflow, cap, shape);
        case 16: return launch_t<NW, 16>(P, s_lv, sb, num_sms, stream, overflow, cap, shape);
        case 32: return launch_t<NW, 32>(P, s_lv, sb, num_sms, stream, overflow, cap, shape);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_genasm(const KernelParams& P, int group, int s_lv, int sb, int num_sms,
                          cudaStream_t stream, uint32_t** overflow, size_t* cap,
                          LaunchShape* shape) {
    if (P.W <= 32) return launch_nw<1>(P, group, s_lv, sb, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_nw<2>(P, group, s_lv, sb, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_nw<4>(P, group, s_lv, sb, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm
