// genasm_baseline.cu -- the unimproved GenASM engine (mode="baseline") on sm_100a.
//
// The reference's dense engine (dc_baseline, pkg/src/bitalign/distance.py:153-218,
// table BaselineEdgeTable, dptable.py:195-247, traceback over stored edges,
// backtrace.py:100-111): every window computes ALL k+1 levels and stores the
// four edge vectors (M, S, D, I) of every entry -- 4 (k+1) n rows of
// ceil(m/64) words -- and the traceback reads edges instead of recomputing
// them.  It gives the same alignments as the improved engine and differs in
// the counters (rows_computed = k+1 per window, entry_writes = 4 (k+1) n,
// 1 or 4 reads per traceback step), which is what it exists to measure: the
// improved-vs-unimproved ratios of the paper on the same device.
//
// One warp per pair, pairs from the global queue.  DC: a levels-as-lanes
// wavefront (lane q owns level 32p+q of pass p, full-width rows of NW 64-bit
// words, R[d-1][j] from lane q-1 by shuffle, the last level of a pass handed
// to the next pass through a carry row buffer); the edges go to the warp's
// dense table in global memory, [column][level][edge][word].  TB: lane 0
// walks the stored edges.
#include "genasm_kernel.cuh"

namespace genasm {

namespace {

constexpr int kBBlock = 128;
constexpr int kBWarps = kBBlock / 32;
constexpr unsigned FULLM = 0xffffffffu;

template <int NW>
struct Row {
    uint64_t w[NW];
};

template <int NW>
__device__ __forceinline__ Row<NW> sh1(const Row<NW>& x) {  // toward higher bits, 0 in
    Row<NW> r;
#pragma unroll
    for (int u = NW - 1; u > 0; --u) r.w[u] = (x.w[u] << 1) | (x.w[u - 1] >> 63);
    r.w[0] = x.w[0] << 1;
    return r;
}

template <int NW>
__device__ __forceinline__ Row<NW> init_row(int m, int d) {  // bits < min(d, m) are 0
    const int z = d < m ? d : m;
    Row<NW> r;
#pragma unroll
    for (int u = 0; u < NW; ++u) {
        const int lo = 64 * u;
        r.w[u] = z <= lo ? ~0ull : (z >= lo + 64 ? 0ull : ~0ull << (z - lo));
    }
    return r;
}

template <int NW>
__device__ __forceinline__ Row<NW> shfl_up_row(const Row<NW>& x) {
    Row<NW> r;
#pragma unroll
    for (int u = 0; u < NW; ++u) r.w[u] = __shfl_up_sync(FULLM, x.w[u], 1);
    return r;
}

template <int NW>
__device__ __forceinline__ bool bit0(const Row<NW>& x, int i) {  // bit i is 0 (active)
    return !((x.w[i >> 6] >> (i & 63)) & 1ull);
}

struct BPair {
    int pair, Lp, Lt, widx;
    int64_t pat, txt, ops, dst, t, nops, cost, rows, reads, writes, words;
};

__device__ void bfinish(const KernelParams& P, const BPair& S, int status) {
    PairResult r{};
    r.status = status;
    r.fail_window = status == 0 || status == 2 ? -1 : S.widx;
    if (status == 0) {
        r.cost = S.cost;
        r.text_consumed = S.t;
        r.rows_computed = S.rows;
        r.ops_len = S.nops;
        r.entry_reads = S.reads;
        r.entry_writes = S.writes;
        r.words_allocated = S.words;
    } else if (status != 2) {  // the windows a failed pair never completed read as 0
        const int64_t step = P.W - P.O;
        const int64_t nwin = S.Lp <= P.W ? 1 : 1 + (S.Lp - P.W + step - 1) / step;
        for (int64_t i = S.widx; i < nwin; ++i) P.dists[S.dst + i] = 0;
    }
    reinterpret_cast<PairResult*>(P.results)[S.pair] = r;
}

// one window: all k+1 levels into the dense edge table; returns d_min or -1
template <int NW>
__device__ int dc_dense(const KernelParams& P, int m, int n, const uint8_t* tch, const Row<NW>* pm,
                        uint64_t* tab, uint64_t* carry, int lane) {
    const int K = P.k;
    int dmin = 1 << 30;
    const int passes = (K + 1 + 31) / 32;
    for (int pass = 0; pass < passes; ++pass) {
        const int d = pass * 32 + lane;
        const bool live = d <= K;
        Row<NW> cur = init_row<NW>(m, d);                      // R[d][j-1]
        Row<NW> diag = init_row<NW>(m, d > 0 ? d - 1 : 0);     // R[d-1][j-1]
        Row<NW> out = cur;                                     // this lane's last output
        const uint64_t* cin = carry + (size_t)((pass + 1) & 1) * 128 * NW;  // level 32p-1
        uint64_t* cout = carry + (size_t)(pass & 1) * 128 * NW;
        for (int s = 0; s < n + 31; ++s) {
            Row<NW> up = shfl_up_row<NW>(out);                 // R[d-1][j] from lane q-1
            const int j = s - lane + 1;
            if (live && j >= 1 && j <= n) {
                if (lane == 0 && d > 0) {
#pragma unroll
                    for (int u = 0; u < NW; ++u) up.w[u] = cin[(size_t)(j - 1) * NW + u];
                }
                const Row<NW> p = pm[tch[j - 1]];
                Row<NW> me = sh1<NW>(cur), r;
#pragma unroll
                for (int u = 0; u < NW; ++u) me.w[u] |= p.w[u];
                uint64_t* e = tab + ((size_t)(j - 1) * (K + 1) + d) * 4 * NW;
                if (d == 0) {
                    r = me;
#pragma unroll
                    for (int u = 0; u < NW; ++u) {
                        e[u] = me.w[u];
                        e[NW + u] = e[2 * NW + u] = e[3 * NW + u] = ~0ull;
                    }
                } else {
                    const Row<NW> se = sh1<NW>(diag), ie = sh1<NW>(up);
#pragma unroll
                    for (int u = 0; u < NW; ++u) {
                        r.w[u] = me.w[u] & se.w[u] & diag.w[u] & ie.w[u];
                        e[u] = me.w[u];
                        e[NW + u] = se.w[u];
                        e[2 * NW + u] = diag.w[u];
                        e[3 * NW + u] = ie.w[u];
                    }
                }
                diag = up;
                cur = r;
                out = r;
                if (lane == 31) {
#pragma unroll
                    for (int u = 0; u < NW; ++u) cout[(size_t)(j - 1) * NW + u] = r.w[u];
                }
            }
        }
        // R[d][n] bit m-1 == 0 solves level d (n == 0: the init row)
        const bool ok = live && bit0<NW>(cur, m - 1);
        const unsigned b = __ballot_sync(FULLM, ok);
        if (b && dmin > K) dmin = pass * 32 + __ffs(b) - 1;
        __syncwarp();  // the carry rows of this pass are read by the next
    }
    return dmin <= K ? dmin : -1;
}

template <int NW>
__global__ void __launch_bounds__(kBBlock)
genasm_baseline_kernel(const KernelParams P, uint64_t* scratch, int64_t words_per_warp) {
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint64_t* tab = scratch + gw * words_per_warp;
    uint64_t* carry = tab + (int64_t)(P.k + 1) * P.W * 4 * NW;
    __shared__ uint8_t s_txt[kBWarps][128];
    __shared__ Row<NW> s_pm[kBWarps][5];
    uint8_t* tch = s_txt[wib];
    Row<NW>* pm = s_pm[wib];
    const int W = P.W, K = P.k;
    for (;;) {
        unsigned long long qi = 0;
        if (lane == 0) qi = atomicAdd(P.queue, 1ull);
        qi = __shfl_sync(FULLM, qi, 0);
        if (qi >= (unsigned long long)P.n_pairs) break;
        BPair S{};
        S.pair = P.order ? P.order[qi] : (int)qi;
        S.Lp = P.pat_len[S.pair];
        S.Lt = P.txt_len[S.pair];
        S.pat = P.pat_off[S.pair];
        S.txt = P.txt_off[S.pair];
        S.ops = P.ops_off[S.pair];
        S.dst = P.win_off[S.pair];
        if (S.Lp <= 0) {
            if (lane == 0) bfinish(P, S, 2);  // EmptyPattern (window.py:87-88)
            continue;
        }
        int status = 0;
        for (int64_t p = 0; p < S.Lp;) {  // window.py:95-120
            const int64_t rem = S.Lp - p;
            const bool fin = rem <= W;
            const int m = fin ? (int)rem : W;
            const int64_t tl = S.Lt - S.t;
            const int n = tl < W ? (int)(tl > 0 ? tl : 0) : W;
            const int budget = fin ? m : W - P.O;
            // reversed chunks: pattern bit i = P[p+m-1-i], column j = T[t+n-j]
            __syncwarp();
            for (int x = lane; x < n; x += 32) tch[x] = P.codes[S.txt + S.t + n - 1 - x];
#pragma unroll
            for (int c = 0; c < 5; ++c)
#pragma unroll
                for (int u = 0; u < NW; ++u) {
                    uint64_t w = 0;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = 64 * u + 32 * h + lane;
                        const int sym = i < m ? P.codes[S.pat + p + m - 1 - i] : 4;
                        const unsigned b = __ballot_sync(FULLM, c == 4 || sym != c);
                        w |= (uint64_t)b << (32 * h);
                    }
                    if (lane == 0) pm[c].w[u] = w;
                }
            __syncwarp();
            const int dmin = dc_dense<NW>(P, m, n, tch, pm, tab, carry, lane);
            if (dmin < 0) {
                status = 1;  // WindowFailed(index, k)
                break;
            }
            __syncwarp();
            // traceback over the stored edges (backtrace.py:113-162), lane 0
            int consumed = 0, tcons = 0, wcost = 0;
            if (lane == 0) {
                int j = n, d = dmin, i = m - 1;
                uint8_t* ops = P.ops + S.ops;
                for (;;) {
                    if (i < 0 || consumed >= budget) break;
                    if (j == 0) {
                        if (i + 1 > d) {
                            status = 3;
                            break;
                        }
                        const int take = i + 1 < budget - consumed ? i + 1 : budget - consumed;
                        for (int u = 0; u < take; ++u) ops[S.nops + u] = 'I';
                        S.nops += take;
                        consumed += take;
                        wcost += take;
                        break;
                    }
                    const uint64_t* e = tab + ((size_t)(j - 1) * (K + 1) + d) * 4 * NW;
                    const int wi = i >> 6, bi = i & 63;
                    unsigned mask = ((e[wi] >> bi) & 1ull) ? 0u : 1u;  // M
                    if (d > 0) {
                        mask |= ((e[NW + wi] >> bi) & 1ull) ? 0u : 2u;      // S
                        mask |= ((e[3 * NW + wi] >> bi) & 1ull) ? 0u : 4u;  // I
                        mask |= ((e[2 * NW + wi] >> bi) & 1ull) ? 0u : 8u;  // D
                        S.reads += 4;
                    } else {
                        S.reads += 1;
                    }
                    const int op = (int)((P.prio_lut >> (4 * mask)) & 0xFu);
                    if (op == 0) {
                        ops[S.nops++] = '=';
                        --j, --i, ++consumed, ++tcons;
                    } else if (op == 1) {
                        ops[S.nops++] = 'X';
                        --j, --d, --i, ++consumed, ++tcons, ++wcost;
                    } else if (op == 2) {
                        ops[S.nops++] = 'I';
                        --d, --i, ++consumed, ++wcost;
                    } else if (op == 3) {
                        ops[S.nops++] = 'D';
                        --j, --d, ++tcons, ++wcost;
                    } else {
                        status = 3;  // StuckTraceback
                        break;
                    }
                }
                if (status == 0) {
                    P.dists[S.dst + S.widx] = (uint8_t)dmin;
                    S.rows += K + 1;
                    S.cost += wcost;
                    S.t += tcons;
                    const int64_t wr = 4ll * (K + 1) * n;
                    S.writes += wr;
                    S.words += wr * ((m + 63) / 64);
                }
            }
            status = __shfl_sync(FULLM, status, 0);
            if (status) break;
            S.t = (int64_t)__shfl_sync(FULLM, (unsigned long long)S.t, 0);
            consumed = __shfl_sync(FULLM, consumed, 0);
            ++S.widx;
            p += consumed;
        }
        if (lane == 0) bfinish(P, S, status);
    }
}

}  // namespace

cudaError_t launch_genasm_baseline(KernelParams P, int num_sms, cudaStream_t stream,
                                   uint64_t** scratch, size_t* cap, LaunchShape* shape) {
    const int NW = (P.W + 63) / 64;
    const int per_sm = 4;  // blocks of 4 warps: 16 warps per SM
    int grid = num_sms * per_sm;
    const int64_t warps_needed = P.n_pairs;
    if ((int64_t)grid * kBWarps > warps_needed) grid = (int)((warps_needed + kBWarps - 1) / kBWarps);
    if (grid < 1) grid = 1;
    const int64_t words_per_warp = (int64_t)(P.k + 1) * P.W * 4 * NW + 2 * 128 * NW;
    const size_t need = (size_t)grid * kBWarps * (size_t)words_per_warp;
    cudaError_t e;
    if (need > *cap || !*scratch) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *cap = 0;
        if ((e = cudaMalloc(scratch, need * 8))) return e;
        *cap = need;
    }
    if (NW == 1)
        genasm_baseline_kernel<1><<<grid, kBBlock, 0, stream>>>(P, *scratch, words_per_warp);
    else
        genasm_baseline_kernel<2><<<grid, kBBlock, 0, stream>>>(P, *scratch, words_per_warp);
    if (shape) {
        shape->grid = grid;
        shape->block = kBBlock;
        shape->smem_bytes = 0;
        shape->group = 32;
        shape->blocks_per_sm = per_sm;
        shape->overflow_words_per_group = words_per_warp;
        shape->launches = 1;
    }
    return cudaGetLastError();
}

}  // namespace genasm
