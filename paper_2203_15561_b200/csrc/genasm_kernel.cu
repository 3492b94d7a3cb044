// genasm_kernel.cu -- fused windowed GenASM-DC + GenASM-TB kernel (sm_100a).
// Design summary in genasm_kernel.cuh; roofline and layout in DESIGN.md.
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

// One lane of the DC wavefront: level d = pass*G + q; at step s it evaluates
// column j = s-q+1 of R[d] (distance.py:125-149), receiving R[d-1][j] from
// lane q-1 by shuffle (lane 0: the carry row of the previous pass).
// PRED: fill/drain steps where some lanes are outside [1, n]; MIXED: some
// group of the warp stores full-width rows (full mode) this round.
template <int NW, int G>
struct DcLane {
    using GE = Geo<NW>;
    uint32_t v[NW], a[NW], outv[NW];
    uint32_t lvl0;
    int q, n, amt_base;
    bool active, lane0carry, lastlane, full;
    uint32_t* trow;
    uint32_t* grow;
    uint32_t* crow;
    const uint32_t* prow;

    __device__ __forceinline__ void init(int q_, bool in_dc, int pass, int m, int n_, int K, int W,
                                         bool full_, uint32_t* tab, uint32_t* carry,
                                         const uint32_t* pmcol, uint32_t* gtab) {
        q = q_;
        n = n_;
        const int d = pass * G + q;
        active = in_dc && d <= K;
        lane0carry = active && q == 0 && d > 0;
        lastlane = active && q == G - 1;
        full = full_;
        init_row<NW>(v, m, d);                // R[d][0] = init(m, d)
        init_row<NW>(a, m, d > 0 ? d - 1 : 0);  // R[d-1][0]
        lvl0 = d == 0 ? 0xffffffffu : 0u;     // level 0 has only the match edge
#pragma unroll
        for (int w = 0; w < NW; ++w) outv[w] = 0u;
        amt_base = m - n - 15 - q;            // band origin of column j = s-q+1
        const int dd = d < GE::LV ? d : 0;
        trow = tab + dd * GE::WMAX;
        grow = gtab + (int64_t)d * W * NW;
        crow = carry;
        prow = pmcol;
    }

    template <bool PRED, bool MIXED>
    __device__ __forceinline__ void step(int s) {
        uint32_t b[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) b[w] = __shfl_up_sync(0xffffffffu, outv[w], 1, G);
        const int c = s - q;  // column j-1
        const bool inr = PRED ? (active && (unsigned)c < (unsigned)n) : active;
        if (lane0carry && (!PRED || inr)) {
#pragma unroll
            for (int w = 0; w < NW; ++w) b[w] = crow[c * NW + w];
        }
        uint32_t tt[NW], st[NW], sv[NW], r[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) tt[w] = a[w] & b[w];
        shl1<NW>(tt, st);
        shl1<NW>(v, sv);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t pm = prow[c * NW + w];
            r[w] = (sv[w] | pm) & ((st[w] & a[w]) | lvl0);
        }
        if (!PRED || inr) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                a[w] = b[w];
                v[w] = r[w];
                outv[w] = r[w];
            }
        }
        if (inr) {
            if (!GE::BAND) {
                trow[c] = r[0];
            } else if (MIXED && full) {
#pragma unroll
                for (int w = 0; w < NW; ++w) grow[c * NW + w] = r[w];
            } else {
                int amt = amt_base + s;
                amt = amt < 0 ? 0 : amt;
                if (NW > 2) amt = amt > GE::BAND_MAX ? GE::BAND_MAX : amt;
                trow[c] = band32<NW>(r, amt);
            }
        }
        if (lastlane && (!PRED || inr)) {
#pragma unroll
            for (int w = 0; w < NW; ++w) crow[c * NW + w] = r[w];
        }
    }
};

template <int NW, int G>
__global__ void __launch_bounds__(kMaxBlock)
genasm_kernel(const KernelParams P) {
    using GE = Geo<NW>;
    constexpr int WMAX = GE::WMAX;
    constexpr bool BAND = GE::BAND;
    constexpr int LV = GE::LV;
    extern __shared__ uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int q = lane & (G - 1);
    const int gbase = lane & ~(G - 1);
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
    const unsigned lowmask = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
    const int gib = threadIdx.x / G;
    const int groups_per_block = blockDim.x / G;

    uint32_t* tab = smem + gib * GE::GROUP_W;
    uint32_t* carry = tab + GE::TAB_W;
    uint32_t* pmcol = carry + WMAX * NW;
    uint8_t* cp = reinterpret_cast<uint8_t*>(pmcol + WMAX * NW);
    uint8_t* ct = cp + WMAX;
    const int64_t gid = (int64_t)blockIdx.x * groups_per_block + gib;
    uint32_t* gtab = P.overflow + gid * P.overflow_words_per_group;
    const int W = P.W, O = P.O, K = P.k;
    PairResult* results = reinterpret_cast<PairResult*>(P.results);

    // ---- group-uniform state ----
    int phase = NEED_PAIR;
    int64_t pair = 0;
    int Lp = 0, Lt = 0;
    const uint8_t* Pp = nullptr;
    const uint8_t* Tp = nullptr;
    uint8_t* ops = nullptr;
    uint8_t* dists = nullptr;
    int64_t p = 0, t = 0, nops = 0;
    int widx = 0, m = 0, n = 0, budget = 0, pass = 0, d_min = -1;
    bool full = false;
    // per-pair accumulators (meaningful in lane q == 0)
    int64_t cost = 0, rows = 0, reads = 0, writes = 0, words = 0;

    auto write_result = [&](int status, int fail_window) {
        if (q == 0) {
            PairResult r{};
            r.status = status;
            r.fail_window = fail_window;
            if (status == 0) {
                r.cost = cost;
                r.text_consumed = t;
                r.rows_computed = rows;
                r.ops_len = nops;
                r.entry_reads = reads;
                r.entry_writes = writes;
                r.words_allocated = words;
            }
            results[pair] = r;
        }
    };

    // bit x of table entry (e, col), col >= 1; sets oob if outside the stored band
    auto tbit = [&](int e, int col, int x, bool& oob) -> uint32_t {
        if (BAND && full) {
            const uint32_t* row = gtab + ((int64_t)e * W + (col - 1)) * NW;
            return (row[x >> 5] >> (x & 31)) & 1u;
        }
        const uint32_t word = tab[e * WMAX + (col - 1)];
        if (!BAND) return (word >> x) & 1u;
        int amt = m - 1 - n + col - 15;
        amt = amt < 0 ? 0 : (amt > GE::BAND_MAX ? GE::BAND_MAX : amt);
        const int rel = x - amt;
        if (rel < 0 || rel > 31) {
            oob = true;
            return 1u;
        }
        return (word >> rel) & 1u;
    };

    for (;;) {
        // ================= setup: next pair / next window =================
        while (phase == NEED_PAIR || phase == NEED_WINDOW) {
            if (phase == NEED_PAIR) {
                unsigned long long idx = 0;
                if (q == 0) idx = atomicAdd(P.queue, 1ull);
                idx = __shfl_sync(gmask, idx, 0, G);
                if (idx >= (unsigned long long)P.n_pairs) {
                    phase = DONE;
                    break;
                }
                pair = P.order ? (int64_t)P.order[idx] : (int64_t)idx;
                Lp = P.pat_len[pair];
                Lt = P.txt_len[pair];
                Pp = P.codes + P.pat_off[pair];
                Tp = P.codes + P.txt_off[pair];
                ops = P.ops + P.ops_off[pair];
                dists = P.dists + P.win_off[pair];
                p = t = nops = 0;
                widx = 0;
                cost = rows = reads = writes = words = 0;
                if (Lp <= 0) {  // EmptyPattern (window.py:87-88)
                    write_result(2, -1);
                    continue;
                }
                phase = NEED_WINDOW;
            }
            // ---- window geometry (window.py:96-101) ----
            const int64_t remaining = Lp - p;
            const bool final_w = remaining <= W;
            m = final_w ? (int)remaining : W;
            const int64_t tleft = Lt - t;
            n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
            budget = final_w ? m : W - O;
            // ---- reversed chunks (window.py:99-100) ----
            __syncwarp(gmask);
            for (int i = q; i < m; i += G) cp[i] = Pp[p + m - 1 - i];
            for (int j = q; j < n; j += G) ct[j] = Tp[t + n - 1 - j];
            __syncwarp(gmask);
            // ---- pattern masks (distance.py:70-79), per-column masks (:91-94) ----
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
            pass = 0;
            full = false;
            if (n == 0) {  // R[d][0] = init(m, d) solves iff d >= m
                if (m <= K) {
                    d_min = m;
                    phase = IN_TB;
                } else {
                    write_result(1, widx);
                    phase = NEED_PAIR;
                }
            } else {
                phase = IN_DC;
            }
        }
        if (__all_sync(0xffffffffu, phase == DONE)) break;
        __syncwarp();

        // ================= DC pass round (all groups in lock-step) =================
        {
            const bool in_dc = phase == IN_DC;
            DcLane<NW, G> L;
            L.init(q, in_dc, pass, m, n, K, W, full, tab, carry, pmcol, gtab);
            // warp-uniform trip counts: fill [0, G-1), steady [G-1, nmin), drain [.., steps)
            const int steps = __reduce_max_sync(0xffffffffu, in_dc ? n + G - 1 : 0);
            const int nmin = __reduce_min_sync(0xffffffffu, in_dc ? n : WMAX);
            const int fill_end = steps < G - 1 ? steps : G - 1;
            const int steady_end = nmin > fill_end ? nmin : fill_end;
            if (BAND && __any_sync(0xffffffffu, in_dc && full)) {
                for (int s = 0; s < fill_end; ++s) L.template step<true, true>(s);
                for (int s = fill_end; s < steady_end; ++s) L.template step<false, true>(s);
                for (int s = steady_end; s < steps; ++s) L.template step<true, true>(s);
            } else {
                for (int s = 0; s < fill_end; ++s) L.template step<true, false>(s);
#pragma unroll 4
                for (int s = fill_end; s < steady_end; ++s) L.template step<false, false>(s);
                for (int s = steady_end; s < steps; ++s) L.template step<true, false>(s);
            }
            const bool succ = L.active && n >= 1 &&
                              (word_sel<NW>(L.v, (m - 1) >> 5) & (1u << ((m - 1) & 31))) == 0u;
            if (in_dc) {
                const unsigned bal = (__ballot_sync(gmask, succ) >> gbase) & lowmask;
                if (bal) {
                    d_min = pass * G + __ffs(bal) - 1;
                    phase = IN_TB;
                } else if ((pass + 1) * G > K) {  // NotFound(k) -> WindowFailed(index, k)
                    write_result(1, widx);
                    phase = NEED_PAIR;
                } else if (BAND && !full && (pass + 1) * G >= LV) {
                    full = true;  // d_min > 15: the band cannot serve TB; redo full width
                    pass = 0;
                } else {
                    ++pass;
                }
            }
        }

        // ================= TB round (groups whose window solved) =================
        if (__any_sync(0xffffffffu, phase == IN_TB)) {
            if (phase == IN_TB) {
                __syncwarp(gmask);
                int d = d_min, j = n, i = m - 1, consumed = 0, tcons = 0, wcost = 0;
                int64_t wreads = 0;
                bool stuck = false;
                for (;;) {
                    if (i < 0 || consumed >= budget) break;
                    if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
                        if (i + 1 > d) {
                            stuck = true;
                            break;
                        }
                        const int take = (i + 1 < budget - consumed) ? i + 1 : budget - consumed;
                        for (int u = q; u < take; u += G) ops[nops + u] = 'I';
                        nops += take;
                        wcost += take;
                        consumed += take;
                        i -= take;
                        break;
                    }
                    // lane q evaluates the state q diagonal ('=') steps ahead
                    const int jq = j - q, iq = i - q;
                    int op = OP_STOP, rd = 0;
                    if (iq >= 0 && consumed + q < budget && jq >= 1) {
                        bool oob = false;
                        const int tc = ct[jq - 1];
                        const bool symeq = tc < 4 && cp[iq] == tc;
                        bool mok;
                        if (iq == 0) mok = symeq;
                        else if (jq == 1) mok = symeq && (iq - 1 < d);
                        else mok = symeq && !tbit(d, jq - 1, iq - 1, oob);
                        rd = jq >= 2;
                        bool sok = false, dok = false, iok = false;
                        if (d > 0) {
                            if (jq == 1) {
                                sok = iq == 0 || iq - 1 < d - 1;
                                dok = iq < d - 1;
                            } else {
                                sok = iq == 0 || !tbit(d - 1, jq - 1, iq - 1, oob);
                                dok = !tbit(d - 1, jq - 1, iq, oob);
                                rd += 1;
                            }
                            iok = iq == 0 || !tbit(d - 1, jq, iq - 1, oob);
                            rd += 1;
                        }
                        op = OP_STUCK;
#pragma unroll
                        for (int u = 3; u >= 0; --u) {
                            const int id = (P.prio >> (2 * u)) & 3;
                            const bool ok = id == OP_M ? mok : id == OP_S ? sok : id == OP_I ? iok : dok;
                            if (ok) op = id;
                        }
                        if (oob) op = OP_STUCK;
                    }
                    const unsigned nz = (__ballot_sync(gmask, op != OP_M) >> gbase) & lowmask;
                    const int f = nz ? __ffs(nz) - 1 : G;
#ifdef GA_DEBUG
                    if (pair == 1)
                        printf("TB q=%d state d=%d j=%d i=%d c=%d -> lane (jq=%d iq=%d) op=%d f=%d\n", q,
                               d, j, i, consumed, jq, iq, op, f);
#endif
                    if (q < f) ops[nops + q] = '=';
                    wreads += __reduce_add_sync(gmask, q < f ? (unsigned)rd : 0u);
                    j -= f;
                    i -= f;
                    consumed += f;
                    tcons += f;
                    nops += f;
                    if (f == G) continue;
                    const int opf = __shfl_sync(gmask, op, f, G);
                    const int rdf = __shfl_sync(gmask, rd, f, G);
                    if (opf == OP_STOP) continue;
                    if (opf == OP_STUCK) {
                        stuck = true;
                        break;
                    }
                    wreads += rdf;
                    uint8_t ch;
                    if (opf == OP_S) {
                        ch = 'X'; --j; --d; --i; ++consumed; ++tcons;
                    } else if (opf == OP_I) {
                        ch = 'I'; --d; --i; ++consumed;
                    } else {
                        ch = 'D'; --j; --d; ++tcons;
                    }
                    ++wcost;
                    if (q == 0) ops[nops] = ch;
                    ++nops;
                }
                // entry_writes / words_allocated of this window in closed form
                // (sum over stored columns per level, dptable.py:62-82, 156-171)
                unsigned wr = 0;
                for (int dd = q; dd <= d_min; dd += G) {
                    int ss = n - budget - (K - dd) - 1;
                    ss = ss > 1 ? ss : 1;
                    const int cnt = n - ss + 1;
                    wr += cnt > 0 ? (unsigned)cnt : 0u;
                }
                wr = __reduce_add_sync(gmask, wr);
                if (stuck) {
                    write_result(3, widx);
                    phase = NEED_PAIR;
                } else {
                    if (q == 0) {
                        dists[widx] = (uint8_t)d_min;
                        rows += d_min + 1;
                        cost += wcost;
                        reads += wreads;
                        writes += wr;
                        words += (int64_t)wr * ((m + 63) / 64);
                    }
                    p += consumed;
                    t += tcons;
                    ++widx;
                    if (p < Lp) {
                        phase = NEED_WINDOW;
                    } else {
                        write_result(0, -1);
                        phase = NEED_PAIR;
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------

template <int NW, int G>
static cudaError_t launch_t(const KernelParams& base, int block, int num_sms, cudaStream_t stream,
                            uint32_t** overflow, size_t* overflow_cap, LaunchShape* shape) {
    using GE = Geo<NW>;
    KernelParams P = base;
    if (block < G || block > kMaxBlock || block % 32) block = 64;
    const int groups_per_block = block / G;
    const int smem = groups_per_block * GE::GROUP_W * 4;
    auto kern = genasm_kernel<NW, G>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int grid = num_sms * per_sm;
    const int64_t max_useful = (P.n_pairs + groups_per_block - 1) / groups_per_block;
    if (grid > max_useful) grid = (int)(max_useful > 0 ? max_useful : 1);
    const int levels_cap = ((P.k + 1 + G - 1) / G) * G;
    P.overflow_words_per_group = GE::BAND ? (int64_t)levels_cap * P.W * NW : 0;
    const size_t need = (size_t)grid * groups_per_block * (size_t)P.overflow_words_per_group;
    if (need > *overflow_cap || !*overflow) {
        if (*overflow) cudaFree(*overflow);
        *overflow = nullptr;
        *overflow_cap = 0;
        e = cudaMalloc(overflow, need * 4 + 64);
        if (e != cudaSuccess) return e;
        *overflow_cap = need;
    }
    P.overflow = *overflow;
    kern<<<grid, block, smem, stream>>>(P);
    shape->grid = grid;
    shape->block = block;
    shape->smem_bytes = smem;
    shape->group = G;
    shape->blocks_per_sm = per_sm;
    shape->overflow_words_per_group = P.overflow_words_per_group;
    return cudaGetLastError();
}

template <int NW>
static cudaError_t launch_nw(const KernelParams& P, int group, int block, int num_sms,
                             cudaStream_t stream, uint32_t** overflow, size_t* cap,
                             LaunchShape* shape) {
    switch (group) {
        case 8: return launch_t<NW, 8>(P, block, num_sms, stream, overflow, cap, shape);
        case 16: return launch_t<NW, 16>(P, block, num_sms, stream, overflow, cap, shape);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_genasm(const KernelParams& P, int group, int block, int num_sms,
                          cudaStream_t stream, uint32_t** overflow, size_t* cap,
                          LaunchShape* shape) {
    if (P.W <= 32) return launch_nw<1>(P, group, block, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_nw<2>(P, group, block, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_nw<4>(P, group, block, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm
