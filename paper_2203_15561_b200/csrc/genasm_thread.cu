// genasm_thread.cu -- lane-per-pair fused DC+TB kernel (sm_100a), W <= 64.
//
// Every lane owns one pair and walks its window chain (window.py:95-120)
// alone: DC in 32-bit diagonal bands (16 levels, exact for d_min <= 15; see
// genasm_thread.cuh), traceback from the lane's own band table, next window.
// No shuffles or cross-lane waits on the hot loop: four 32-bit operations
// per DC entry.
//
// Windows with d_min > 15 (a few percent at 10 % divergence) need the full
// tier (full-width rows, 16-level passes).  A lane that meets one parks the
// pair (state saved in its result record, id pushed on the warp's HARD stack
// in shared memory) and takes another pair, so the warp's fast loop never
// diverges into the slow path.  When 32 hard windows are parked (or nothing
// else is left) the warp runs them together: active pairs are parked on the
// RESUME stack, each lane runs one hard window, the pairs go back on RESUME,
// and free lanes refill from RESUME before taking fresh pairs from the warp's
// static share of the longest-first order (dealt round-robin across warps).  Parked pairs resume oldest first, and while pairs
// wait the active ones rotate out every 8 windows: every pair of a warp
// advances at the same pace, so the warp's pairs finish together.
//
// Tables.  Band tier: per warp, [column][word quad][lane] x 16 B -- each
// column's 16 levels are 8 paired words (genasm_thread.cuh), two coalesced
// 16-byte stores per lane.  Full tier: per lane,
// [level][column] x 8 B.  Both live in the context's scratch slab.
#include "genasm_device.cuh"
#include "genasm_thread.cuh"

namespace genasm {

#ifdef GA_THREAD_STATS
// dev counters: band steps, active lanes summed over band steps, hard batches,
// hard lanes summed over batches
__device__ unsigned long long g_thread_stats[8];
#define GA_STAT(k, v) (lane == 0 ? (void)atomicAdd(&g_thread_stats[k], (unsigned long long)(v)) : (void)0)
#else
#define GA_STAT(k, v) ((void)0)
#endif

namespace {

constexpr int kTBlock = 128;           // threads per block
constexpr int kWarps = kTBlock / 32;
constexpr int kStack = 128;            // per-warp HARD / RESUME stack entries
constexpr int kHandoff = 24;           // full-tier windows before a pair is handed over
constexpr int kBandWordsPerWarp = 64 * 2 * 32 * 4;  // W <= 64 columns x 8 paired words x 32 lanes

struct BandTab {
    uint4* base;  // this warp's region: [column][word quad][lane] x 16 B
    int lane;
    __device__ __forceinline__ void put(int j, const uint32_t* w) {
        uint4* p = base + (size_t)(j - 1) * 64 + lane;
        p[0] = make_uint4(w[0], w[1], w[2], w[3]);
        p[32] = make_uint4(w[4], w[5], w[6], w[7]);
    }
    __device__ __forceinline__ uint32_t get(int k, int c) const {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(base + (size_t)(c - 1) * 64 +
                                                              (k >> 2) * 32 + lane);
        return p[k & 3];
    }
};

struct FullTab {
    uint64_t* base;  // this lane's rows, [column 1..W][level 0..LV)
    int LV;
    __device__ __forceinline__ void put4(int d0, int j, const uint32_t* lo, const uint32_t* hi) {
        uint4* p = reinterpret_cast<uint4*>(base + (size_t)(j - 1) * LV + d0);
        p[0] = make_uint4(lo[0], hi[0], lo[1], hi[1]);
        p[1] = make_uint4(lo[2], hi[2], lo[3], hi[3]);
    }
    __device__ __forceinline__ uint64_t get(int d, int j) const {
        return base[(size_t)(j - 1) * LV + d];
    }
};

// full-tier rows stored per column: levels 0..k rounded up to whole passes
__host__ __device__ __forceinline__ int full_levels(int k) {
    return (k + thr::kPassLevels) / thr::kPassLevels * thr::kPassLevels;
}

// per-lane pair state (between windows)
struct Lane {
    int pair;  // -1: none
    int Lp, Lt, widx, hardc;  // hardc: windows that needed the full tier
    int64_t pat, txt, ops, dst;  // offsets
    int64_t t, nops, cost, rows, reads, writes, words;
};

__device__ __forceinline__ void open_pair(const KernelParams& P, Lane& L, int pair) {
    L.pair = pair;
    L.Lp = P.pat_len[pair];
    L.Lt = P.txt_len[pair];
    L.pat = P.pat_off[pair];
    L.txt = P.txt_off[pair];
    L.ops = P.ops_off[pair];
    L.dst = P.win_off[pair];
}

__device__ __forceinline__ void fresh_pair(const KernelParams& P, Lane& L, int pair) {
    open_pair(P, L, pair);
    L.widx = 0;
    L.hardc = 0;
    L.t = L.nops = L.cost = L.rows = L.reads = L.writes = L.words = 0;
}

// park: the running state goes into the pair's own result record
__device__ __forceinline__ void park(const KernelParams& P, const Lane& L) {
    PairResult* r = reinterpret_cast<PairResult*>(P.results) + L.pair;
    r->status = -1 - L.hardc;
    r->fail_window = L.widx;
    r->cost = L.cost;
    r->text_consumed = L.t;
    r->rows_computed = L.rows;
    r->ops_len = L.nops;
    r->entry_reads = L.reads;
    r->entry_writes = L.writes;
    r->words_allocated = L.words;
}

__device__ __forceinline__ void unpark(const KernelParams& P, Lane& L, int pair) {
    open_pair(P, L, pair);
    const PairResult* r = reinterpret_cast<const PairResult*>(P.results) + pair;
    L.hardc = -1 - r->status;
    L.widx = r->fail_window;
    L.cost = r->cost;
    L.t = r->text_consumed;
    L.rows = r->rows_computed;
    L.nops = r->ops_len;
    L.reads = r->entry_reads;
    L.writes = r->entry_writes;
    L.words = r->words_allocated;
}

__device__ __forceinline__ void finish(const KernelParams& P, Lane& L, int status) {
    PairResult r{};
    r.status = status;
    r.fail_window = -1;
    if (status == 0) {
        r.cost = L.cost;
        r.text_consumed = L.t;
        r.rows_computed = L.rows;
        r.ops_len = L.nops;
        r.entry_reads = L.reads;
        r.entry_writes = L.writes;
        r.words_allocated = L.words;
    } else if (status != 2) {
        r.fail_window = L.widx;
        // windows the pair never completed read as 0
        const int64_t step = P.W - P.O;
        const int64_t nwin = L.Lp <= P.W ? 1 : 1 + (L.Lp - P.W + step - 1) / step;
        for (int64_t i = L.widx; i < nwin; ++i) P.dists[L.dst + i] = 0;
    }
    reinterpret_cast<PairResult*>(P.results)[L.pair] = r;
    L.pair = -1;
}

enum : int { WIN_NEXT = 0, WIN_HARD = 1 };

// One window of lane L's pair.  FULL = false: band tier, returns WIN_HARD if
// d_min > 15 (and k allows more); FULL = true: full tier.  On completion of
// the pair (or failure) the result is written and L.pair = -1.
template <bool FULL>
__device__ __forceinline__ int run_window(const KernelParams& P, Lane& L, BandTab& bt, FullTab& ft) {
    using namespace thr;
    const int W = P.W, K = P.k;
    const int64_t p = (int64_t)L.widx * (W - P.O);  // every earlier window consumed W-O
    const int64_t rem = L.Lp - p;
    const bool fin = rem <= W;
    const int m = fin ? (int)rem : W;
    const int64_t tl = L.Lt - L.t;
    const int n = tl < W ? (int)(tl > 0 ? tl : 0) : W;
    const int budget = fin ? m : W - P.O;
    const Planes pp = load_planes_bits(P.planes, P.plane_words, L.pat + p, m);
    Planes tp{0ull, 0ull, 0ull};
    int d_min;
    uint8_t* ops = P.ops + L.ops;
    TbOut o;
    bool ok;
    if (n == 0) {  // R[d][0] = init(m, d) solves iff d >= m
        if (m > K) {
            finish(P, L, 1);
            return WIN_NEXT;
        }
        d_min = m;
        ok = traceback([&](int, int, int) -> uint32_t { return 1u; }, pp, tp, m, n, d_min, budget,
                       P.prio_lut, ops, L.nops, o);
    } else {
        tp = load_planes_bits(P.planes, P.plane_words, L.txt + L.t, n);
        if (!FULL) {
            uint32_t okm = dc_band(pp, tp, m, n, bt);
            const int lim = K < 15 ? K : 15;
            okm &= (2u << lim) - 1u;
            if (!okm) {
                if (K <= 15) {
                    finish(P, L, 1);
                    return WIN_NEXT;
                }
                return WIN_HARD;
            }
            d_min = __ffs(okm) - 1;
            ok = tb_band(bt, pp, tp, m, n, d_min, budget, P.prio_lut, ops, L.nops, o);
        } else {
            d_min = dc_full(pp, tp, m, n, K, ft);
            if (d_min < 0) {
                finish(P, L, 1);
                return WIN_NEXT;
            }
            ok = traceback([&](int e, int c, int x) { return full_bit(ft, e, c, x); }, pp, tp, m, n,
                           d_min, budget, P.prio_lut, ops, L.nops, o);
        }
    }
    if (!ok) {
        finish(P, L, 3);
        return WIN_NEXT;
    }
    const int64_t wr = window_writes(n, budget, K, d_min);
    P.dists[L.dst + L.widx] = (uint8_t)d_min;
    L.rows += d_min + 1;
    L.cost += o.wcost;
    L.reads += o.reads;
    L.writes += wr;
    L.words += wr * ((m + 63) / 64);
    L.t += o.tcons;
    ++L.widx;
    if (p + o.consumed >= L.Lp) finish(P, L, 0);
    return WIN_NEXT;
}

// One full-tier window of a parked pair.  Returns true if the pair goes back
// on RESUME.
__device__ __forceinline__ bool hard_window(const KernelParams& P, int pair, uint4* band, int lane,
                                         uint64_t* full) {
    Lane L;
    unpark(P, L, pair);
    BandTab bt{band, lane};
    FullTab ft{full, full_levels(P.k)};
    run_window<true>(P, L, bt, ft);
    if (L.pair < 0) return false;
    park(P, L);
    return true;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

}  // namespace

// codes -> three bit-planes: thread t packs symbols [64t, 64t+64) of each
// plane into one 64-bit word (bit 0 of the code, bit 1, code 4)
__global__ void __launch_bounds__(256) planes_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                     uint64_t* __restrict__ pl, int64_t words) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < words;
         t += (int64_t)gridDim.x * blockDim.x) {
        uint64_t f0 = 0, f1 = 0, fn = 0;
        const int64_t s0 = t * 64;
        if (s0 + 64 <= n && ((reinterpret_cast<uintptr_t>(codes) & 15) == 0)) {
            const uint4* q = reinterpret_cast<const uint4*>(codes + s0);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const uint4 x = __ldg(q + v);
                const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int pos = 16 * v + 4 * u;
                    f0 |= (uint64_t)thr::nib(w4[u], 0) << pos;
                    f1 |= (uint64_t)thr::nib(w4[u], 1) << pos;
                    fn |= (uint64_t)thr::nib(w4[u], 2) << pos;
                }
            }
        } else {
            for (int k = 0; k < 64 && s0 + k < n; ++k) {
                const uint8_t c = codes[s0 + k];
                f0 |= (uint64_t)(c & 1) << k;
                f1 |= (uint64_t)((c >> 1) & 1) << k;
                fn |= (uint64_t)((c >> 2) & 1) << k;
            }
        }
        pl[t] = f0;
        pl[words + t] = f1;
        pl[2 * words + t] = fn;
    }
}

#ifndef GA_THREAD_MINB
#define GA_THREAD_MINB 4  // resident blocks per SM the register budget must allow
#endif

__global__ void __launch_bounds__(kTBlock, GA_THREAD_MINB)
genasm_thread_kernel(const KernelParams P, uint32_t* band_base, uint64_t* full_base,
                     int64_t full_words_per_lane) {
    __shared__ int s_hard[kWarps][kStack], s_res[kWarps][kStack];
    __shared__ int s_nh[kWarps], s_rh[kWarps], s_rt[kWarps];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    BandTab bt{reinterpret_cast<uint4*>(band_base + gw * kBandWordsPerWarp), lane};
    FullTab ft{full_base + (gw * 32 + lane) * full_words_per_lane, full_levels(P.k)};
    int* hard = s_hard[wib];  // stack of parked hard windows
    int* res = s_res[wib];    // FIFO ring of parked pairs ready to resume
    if (lane == 0) s_nh[wib] = s_rh[wib] = s_rt[wib] = 0;
    __syncwarp();
    const unsigned lt = lanemask_lt();
    bool exhausted = false;
    int steps = 0;
    int64_t taken = 0;
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    Lane L;
    L.pair = -1;
    for (;;) {
        // ---- free lanes take parked pairs first (oldest first), then fresh ones ----
        unsigned freem = __ballot_sync(FULL, L.pair < 0);
        if (freem) {
            const int rh = s_rh[wib], nr = s_rt[wib] - rh;
            const int rank = __popc(freem & lt);
            const int take = min(__popc(freem), nr);
            if (L.pair < 0 && rank < take) unpark(P, L, res[(rh + rank) & (kStack - 1)]);
            __syncwarp();
            if (lane == 0) s_rh[wib] = rh + take;
            freem = __ballot_sync(FULL, L.pair < 0);
            if (freem && !exhausted) {
                // fresh pairs: this warp's static share of the longest-first
                // order, dealt round-robin (every warp gets the same work)
                const int cnt = __popc(freem);
                const int64_t k0 = taken;
                taken += cnt;
                if ((uint64_t)(gw + taken * nwarps) >= (uint64_t)P.n_pairs) exhausted = true;
                if (L.pair < 0) {
                    const uint64_t idx = (uint64_t)gw + (uint64_t)(k0 + __popc(freem & lt)) * nwarps;
                    if (idx < (uint64_t)P.n_pairs) {
                        const int pair = P.order ? P.order[idx] : (int)idx;
                        fresh_pair(P, L, pair);
                        if (L.Lp <= 0) finish(P, L, 2);  // EmptyPattern (window.py:87-88)
                    }
                }
            }
        }
        __syncwarp();
        const int nh = s_nh[wib];
        const int nr = s_rt[wib] - s_rh[wib];
        const unsigned active = __ballot_sync(FULL, L.pair >= 0);
        if (!active && nh == 0 && nr == 0 && exhausted) break;
        const int nact = __popc(active);

        // parked hard windows run as a batch once 32 wait, or once at least
        // half of the warp's pairs in flight are parked (lanes would idle);
        // every 8 steps with pairs waiting, the active pairs also rotate out so
        // that all pairs of the warp advance at the same pace (no long tail)
        const bool batch = nh >= 32 || (nh > 0 && nh >= nact + nr);
        const bool rotate = !batch && nr > 0 && nact > 0 && (++steps & 7) == 0;
        if (batch || rotate) {
            int rt = s_rt[wib];
            if (L.pair >= 0) {
                park(P, L);
                res[(rt + __popc(active & lt)) & (kStack - 1)] = L.pair;
                L.pair = -1;
            }
            rt += nact;
            int take = 0;
            if (batch) {
                // ---- hard batch: up to 32 full-tier windows, one per lane ----
                take = nh < 32 ? nh : 32;
                GA_STAT(2, 1);
                GA_STAT(3, take);
                int hp = -1;
                if (lane < take) {
                    hp = hard[nh - 1 - lane];
                    if (!hard_window(P, hp, bt.base, lane, ft.base)) hp = -1;
                }
                const unsigned back = __ballot_sync(FULL, hp >= 0);
                if (hp >= 0) res[(rt + __popc(back & lt)) & (kStack - 1)] = hp;
                rt += __popc(back);
            }
            __syncwarp();
            if (lane == 0) {
                s_rt[wib] = rt;
                s_nh[wib] = nh - take;
            }
            __syncwarp();
            continue;
        }
        if (!active) continue;

        // ---- one band-tier window per active lane ----
        GA_STAT(0, 1);
        GA_STAT(1, nact);
        int r = WIN_NEXT;
        if (L.pair >= 0) r = run_window<false>(P, L, bt, ft);
        // a pair whose windows keep needing the full tier (e.g. unrelated
        // sequences) goes to the lane-group kernel instead of the hard stack
        if (r == WIN_HARD && ++L.hardc > kHandoff) {
            park(P, L);
            P.handoff[atomicAdd(P.n_handoff, 1ull)] = L.pair;
            L.pair = -1;
            r = WIN_NEXT;
        }
        const unsigned hm = __ballot_sync(FULL, r == WIN_HARD);
        if (hm) {
            if (r == WIN_HARD) {
                park(P, L);
                hard[nh + __popc(hm & lt)] = L.pair;
                L.pair = -1;
            }
            __syncwarp();
            if (lane == 0) s_nh[wib] = nh + __popc(hm);
            __syncwarp();
        }
    }
}

cudaError_t launch_genasm_thread(const KernelParams& base, int num_sms, cudaStream_t stream,
                                 uint32_t** scratch, size_t* cap, uint32_t** lock_scratch,
                                 size_t* lock_cap, LaunchShape* shape) {
    if (base.W > 64) return cudaErrorInvalidValue;
    KernelParams P = base;
    int per_sm = 0;
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, genasm_thread_kernel, kTBlock, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const char* cap_env = getenv("GA_WARPS_PER_SM");
    const int warps_cap = cap_env && atoi(cap_env) > 0 ? atoi(cap_env) : 16;
    const int bcap = warps_cap / kWarps;
    if (bcap >= 1 && per_sm > bcap) per_sm = bcap;
    // pairs are long sequential chains, so give every lane the same number of
    // pairs: the fewest waves the resident lanes allow, then just enough warps
    const int64_t resident = (int64_t)num_sms * per_sm * kTBlock;
    const int64_t waves = (P.n_pairs + resident - 1) / resident;
    const int64_t lanes = (P.n_pairs + waves - 1) / (waves > 0 ? waves : 1);
    int grid = (int)((lanes + kTBlock - 1) / kTBlock);
    if (grid < 1) grid = 1;
    // scratch: band tables | full-tier rows (W x levels x 8 B per lane) |
    // hand-over list (n_pairs ids) | its counter
    const int64_t full_words = (int64_t)full_levels(P.k) * P.W * 2;
    const size_t warps = (size_t)grid * kWarps;
    const size_t band_words = (warps * kBandWordsPerWarp + 63) & ~(size_t)63;
    const size_t full_total = (warps * 32 * (size_t)full_words + 63) & ~(size_t)63;
    const size_t list_words = ((size_t)P.n_pairs + 63) & ~(size_t)63;
    // bit-planes: one word per 64 symbols per plane, plus one word of slack
    const int64_t pw = (P.codes_len + 63) / 64 + 1;
    const size_t plane_total = ((size_t)pw * 3 * 2 + 63) & ~(size_t)63;
    const size_t need = band_words + full_total + list_words + 64 + plane_total;
    if (need > *cap || !*scratch) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *cap = 0;
        e = cudaMalloc(scratch, need * 4);
        if (e != cudaSuccess) return e;
        *cap = need;
    }
    uint32_t* band = *scratch;
    uint64_t* full = reinterpret_cast<uint64_t*>(*scratch + band_words);
    P.handoff = reinterpret_cast<int32_t*>(*scratch + band_words + full_total);
    P.n_handoff = reinterpret_cast<unsigned long long*>(*scratch + band_words + full_total +
                                                        list_words);
    if ((e = cudaMemsetAsync(P.n_handoff, 0, sizeof(unsigned long long), stream))) return e;
    uint64_t* planes = reinterpret_cast<uint64_t*>(*scratch + band_words + full_total + list_words + 64);
    P.planes = planes;
    P.plane_words = pw;
    {
        const int64_t blocks = (pw + 255) / 256;
        planes_kernel<<<(int)(blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8), 256, 0, stream>>>(
            P.codes, P.codes_len, planes, pw);
        if ((e = cudaGetLastError())) return e;
    }
    genasm_thread_kernel<<<grid, kTBlock, 0, stream>>>(P, band, full, full_words / 2);
    if ((e = cudaGetLastError())) return e;
    // the handed-over pairs: lane-group kernel, resuming from the parked state
    KernelParams R = P;
    R.order = P.handoff;
    R.n_dev = P.n_handoff;
    R.resume = 1;
    // latency-bound: 32-lane groups, 64 levels per pass, few warps per SM so a
    // group's full-width rows stay in L1 for its traceback
    R.full_only = P.W > 32;
    const char* hg = getenv("GA_HANDOFF_GROUP");
    const char* hw = getenv("GA_HANDOFF_WARPS");
    R.warps_per_sm = hw && atoi(hw) > 0 ? atoi(hw) : 4;
    LaunchShape ls{};
    e = launch_genasm_lockstep(R, hg && atoi(hg) > 0 ? atoi(hg) : (R.full_only ? 32 : 8), 0,
                               num_sms, stream, lock_scratch, lock_cap, &ls);
    shape->grid = grid;
    shape->block = kTBlock;
    shape->smem_bytes = 0;
    shape->group = 1;
    shape->blocks_per_sm = per_sm;
    shape->overflow_words_per_group = full_words;
    shape->launches = 3;
    return e;
}

}  // namespace genasm

#ifdef GA_THREAD_STATS
extern "C" void ga_debug_thread_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, genasm::g_thread_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(genasm::g_thread_stats, z, sizeof z);
    }
}
#endif
