// genasm_thread.cu -- lane-per-pair fused DC+TB kernel (sm_100a), W <= 64,
// and its 16-lane-group form for small batches (the latency path, below).
//
// Every lane owns one pair and walks its window chain (window.py:95-120)
// alone: DC in 32-bit diagonal bands (16 levels, exact for d_min <= 15; see
// genasm_thread.cuh), traceback from the lane's own band table, next window.
// No shuffles or cross-lane waits on the hot loop: four 32-bit operations
// per DC entry.
//
// Windows with d_min > 15 (a few percent at 10 % divergence) are computed by
// the whole warp together, right after the band step that found them: lane q
// owns level q (0..31) of full-width rows and the 32 lanes sweep the window
// as a wavefront (n + 31 steps, one shuffle of R[q-1][j] per step), storing
// the rows in the warp's table (further passes of 32 levels as k allows, lane
// 0 reading the row lane 31 stored); the warp traces back together (coop_tb).
//
// Fresh pairs come from a global longest-first queue, the grid fills every SM
// equally.  A pair with 4 consecutive windows beyond the band tier is handed
// over and finished by the warps that run out of pairs.
//
// Tables, per warp, in the context's scratch slab.  Band tier:
// [column][word quad][lane] x 16 B -- each column's 16 levels are 8 paired
// words (genasm_thread.cuh), two coalesced 16-byte stores per lane.  Full
// tier (one window at a time, the same region): [pass][wavefront step][level]
// x 8 B (full_index).  At the end of each step the warp discards its region's
// L2 lines: the tables are dead and need no write-back.
#include "genasm_device.cuh"
#include "genasm_thread.cuh"

namespace genasm {

#ifdef GA_THREAD_STATS
// dev counters: band steps, active lanes summed over band steps, full-tier
// windows, -, clock cycles in band steps, in full-tier windows
__device__ unsigned long long g_thread_stats[18];  // [8]/[9] band DC/TB cycles, [10]/[11] full-tier DC/TB, [12] group window set-up, [14]/[15]/[16] hand-over tail windows, their DC/TB cycles
// per pair: first window started, finished (globaltimer ns), full-tier windows
__device__ unsigned long long g_pair_t[4][262144];  // + [3]: taken from the hand-over list
#define GA_STAT(k, v) (lane == 0 ? (void)atomicAdd(&g_thread_stats[k], (unsigned long long)(v)) : (void)0)
#else
#define GA_STAT(k, v) ((void)0)
#endif

// GA_CHECK: the debug build's contract checks (build.py --check ->
// _genasm_check.so, tests/test_check_build.py).  A violated check records its
// code and source line in g_check (first one kept, all counted) and, where a
// pair is involved, fails that pair as GA_STUCK -- the reference raises
// PrunedAccess for a read of an entry it never stored (dptable.py:20-30,
// raised at :183-184) and StuckTraceback for a walk with no active edge
// (backtrace.py:30-35).  Codes: 1 band-table read outside the stored columns
// or levels (PrunedAccess), 3 a full-tier read outside the columns or levels
// computed, 4 ops beyond the pair's capacity, 5 window distances beyond the
// pair's count, 6 a hand-over entry that is not a pair, 7 a table store
// outside the warp's region.
#ifdef GA_CHECK
__device__ unsigned long long g_check[4];  // [0] first (code << 32 | line), [1] count, [2]/[3] detail
__device__ __noinline__ void ga_check_fail(int code, int line, long long a, long long b) {
    if (atomicCAS(&g_check[0], 0ull, (unsigned long long)code << 32 | (unsigned)line) == 0ull) {
        g_check[2] = (unsigned long long)a;
        g_check[3] = (unsigned long long)b;
    }
    atomicAdd(&g_check[1], 1ull);
}
#define GA_ASSERT(cond, code, a, b) \
    ((cond) ? true : (ga_check_fail((code), __LINE__, (long long)(a), (long long)(b)), false))
#else
#define GA_ASSERT(cond, code, a, b) true
#endif

namespace {

#ifndef GA_TBLOCK
#define GA_TBLOCK 128
#endif
constexpr int kTBlock = GA_TBLOCK;  // threads per block
constexpr int kWarps = kTBlock / 32;
constexpr int kFullLevels = 32;  // full tier: one level per lane
// consecutive full-tier windows before a hand-over: 8 for the lane-per-pair
// launches (config 3 37.1 -> 36.4 ms against 4: a pair over a long indel
// stays in its lane instead of running all its remaining windows on a whole
// warp; 2: 101 ms), 4 for the lane groups (config 5 10.6 ms against 11.1)
constexpr int kStreak = 8;
constexpr int kStreakGroups = 4;
constexpr int kBandWordsPerWarp = 64 * 2 * 32 * 4;  // W <= 64 columns x 8 paired words x 32 lanes

// full-tier table: [pass][wavefront step][level within the pass], 24 KB per
// pass -- entry (d, j) was written at step j-1+(d mod 32) of its pass, so each
// step's 32 rows are one coalesced 256-byte store
__device__ __forceinline__ int full_index(int d, int j) {
    const int e = d & 31;
    return (d >> 5) * (96 * kFullLevels) + (j - 1 + e) * kFullLevels + e;
}

// Band-table columns below n - GA_COLD_COLS are stored with an L2 evict-first
// policy: the traceback (about budget + d_min columns back from n) rarely
// reaches them, and they are the oldest lines when it does, so they should
// leave L2 before the columns every traceback reads.  Measured on config 3:
// 39.1 -> 37.6 ms for 28..46 (all columns evict-first 38.1 ms; the read
// columns evict-last 39.4 ms).  0 disables.
#ifndef GA_COLD_COLS
#define GA_COLD_COLS 40
#endif

__device__ __forceinline__ void st_v4_policy(uint4* p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

struct BandTab {
    uint4* base;  // this warp's region: [column][word quad][lane] x 16 B
    int lane;
#if GA_COLD_COLS
    int jhot;      // columns below jhot: rarely read by the traceback
    uint64_t pol;  // L2 evict-first policy
#endif
#ifdef GA_CHECK
    int jlo, jhi;      // the columns stored this window
    mutable bool bad;  // a read outside them (PrunedAccess)
#endif

    __device__ __forceinline__ void put(int j, const uint32_t* w) {
        if (!GA_ASSERT(j >= 1 && j <= 64, 7, j, 0)) return;
        uint4* p = base + (size_t)(j - 1) * 64 + lane;
#if GA_COLD_COLS
        if (j < jhot) {
            st_v4_policy(p, make_uint4(w[0], w[1], w[2], w[3]), pol);
            st_v4_policy(p + 32, make_uint4(w[4], w[5], w[6], w[7]), pol);
            return;
        }
#endif
        p[0] = make_uint4(w[0], w[1], w[2], w[3]);
        p[32] = make_uint4(w[4], w[5], w[6], w[7]);
    }
    // word k of column c (thr::packed_word(e) holds level e)
    __device__ __forceinline__ uint32_t get(int k, int c) const {
#ifdef GA_CHECK
        if (!GA_ASSERT(c >= jlo && c <= jhi && k >= 0 && k < 8, 1, c, k)) {
            bad = true;
            return 0xffffffffu;
        }
#endif
        const uint32_t* p = reinterpret_cast<const uint32_t*>(base + (size_t)(c - 1) * 64 +
                                                              (k >> 2) * 32 + lane);
        return p[k & 3];
    }
    __device__ __forceinline__ int wi(int e) const { return thr::packed_word(e); }
    __device__ __forceinline__ uint32_t bit(uint32_t w, int e, int b) const {
        return thr::packed_bit(w, e, b);
    }
};

// per-lane pair state (between windows)
struct Lane {
    int pair;  // -1: none
    int Lp, Lt, widx;
    int streak;  // consecutive windows beyond the band tier
    int64_t pat, txt, ops, dst;  // offsets
    int64_t t, nops, cost, rows, reads, writes, words;
};

__device__ __forceinline__ void fresh_pair(const KernelParams& P, Lane& L, int pair) {
    L.pair = pair;
#ifdef GA_THREAD_STATS
    if (pair < 262144) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        atomicMin(&g_pair_t[0][pair], tnow);
    }
#endif
    L.Lp = P.pat_len[pair];
    L.Lt = P.txt_len[pair];
    L.pat = P.pat_off[pair];
    L.txt = P.txt_off[pair];
    L.ops = P.ops_off[pair];
    L.dst = P.win_off[pair];
    L.widx = 0;
    L.streak = 0;
    L.t = L.nops = L.cost = L.rows = L.reads = L.writes = L.words = 0;
}

// a failed pair: its record and the window distances it never completed (0);
// rare, kept out of line
__device__ __noinline__ void fail_pair(PairResult* results, uint8_t* dists, int W, int O, int pair,
                                       int status, int widx, int Lp, int64_t dst) {
    PairResult r{};
    r.status = status;
    r.fail_window = status == 2 ? -1 : widx;
    if (status != 2) {
        const int64_t step = W - O;
        const int64_t nwin = Lp <= W ? 1 : 1 + (Lp - W + step - 1) / step;
        for (int64_t i = widx; i < nwin; ++i) dists[dst + i] = 0;
    }
    results[pair] = r;
}

// The launch parameters are never taken by reference by an out-of-line
// function (fail_pair gets plain values).  A reference makes the compiler keep
// a copy of them in local memory for the whole kernel; with that copy, a
// shared-memory carry added to the full tier's second pass (coop_dc) produced
// wrong window geometry for W = 32, O = 31 -- window_of() saw budget 1 on
// final windows, pairs ran past their pattern -- reproducibly (nvcc 12.9,
// sm_100a; tools/dbg_w32.py), and the same code with values passed was
// correct.  The by-reference form measured 1.5 % faster on config 3; it is not
// worth a code-shape-dependent miscompile (DESIGN 9).
__device__ __forceinline__ void finish(const KernelParams& P, Lane& L, int status) {
    if (status == 0) {
        PairResult r;
        r.status = 0;
        r.fail_window = -1;
        r.cost = L.cost;
        r.text_consumed = L.t;
        r.rows_computed = L.rows;
        r.ops_len = L.nops;
        r.entry_reads = L.reads;
        r.entry_writes = L.writes;
        r.words_allocated = L.words;
        reinterpret_cast<PairResult*>(P.results)[L.pair] = r;
    } else {
        fail_pair(reinterpret_cast<PairResult*>(P.results), P.dists, P.W, P.O, L.pair, status,
                  L.widx, L.Lp, L.dst);
    }
#ifdef GA_THREAD_STATS
    if (L.pair < 262144) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        g_pair_t[1][L.pair] = tnow;
    }
#endif
    L.pair = -1;
}

// geometry of lane L's current window (window.py:96-101)
struct Win {
    int64_t p;
    int m, n, budget;
    bool fin;
};

__device__ __forceinline__ Win window_of(const KernelParams& P, const Lane& L) {
    Win w;
    w.p = (int64_t)L.widx * (P.W - P.O);  // every earlier window consumed W-O
    const int64_t rem = L.Lp - w.p;
    w.fin = rem <= P.W;
    w.m = w.fin ? (int)rem : P.W;
    const int64_t tl = L.Lt - L.t;
    w.n = tl < P.W ? (int)(tl > 0 ? tl : 0) : P.W;
    w.budget = w.fin ? w.m : P.W - P.O;
    return w;
}

// book a finished window (dists, counters, cursors); ends the pair when its
// pattern is consumed
__device__ __forceinline__ void book(const KernelParams& P, Lane& L, const Win& w, int d_min,
                                     const thr::TbOut& o) {
    const int64_t wr = thr::window_writes(w.n, w.budget, P.k, d_min);
#ifdef GA_CHECK
    {
        const int64_t step = P.W - P.O;
        const int64_t nwin = L.Lp <= P.W ? 1 : 1 + (L.Lp - P.W + step - 1) / step;
        GA_ASSERT(L.widx < nwin, 5, L.pair, L.widx);
        GA_ASSERT(L.nops <= (int64_t)L.Lp + L.Lt, 4, L.pair, L.nops);
    }
#endif
    P.dists[L.dst + L.widx] = (uint8_t)d_min;
    L.rows += d_min + 1;
    L.cost += o.wcost;
    L.reads += o.reads;
    L.writes += wr;
    L.words += wr * ((w.m + 63) / 64);
    L.t += o.tcons;
    ++L.widx;
    if (w.p + o.consumed >= L.Lp) finish(P, L, 0);
}

enum : int { WIN_NEXT = 0, WIN_HARD = 1 };

// One band-tier window of lane L's pair.  Returns WIN_HARD (state untouched)
// if d_min > 15 and k allows more; otherwise books the window.
__device__ __forceinline__ int band_window(const KernelParams& P, Lane& L, BandTab& bt) {
    using namespace thr;
    const int K = P.k;
    const Win w = window_of(P, L);
    const Planes pp = load_planes_bits(P.planes, P.plane_words, L.pat + w.p, w.m);
    uint8_t* ops = P.ops + L.ops;
    TbOut o;
    int d_min;
    bool ok;
    if (w.n == 0) {  // R[d][0] = init(m, d) solves iff d >= m
        if (w.m > K) {
            finish(P, L, 1);
            return WIN_NEXT;
        }
        // the walk starts in column 0, whose zeros cover the m insertions
        // (backtrace.py column-0 rule): budget-many 'I'
        d_min = w.m;
        const int take = w.m < w.budget ? w.m : w.budget;
        for (int u = 0; u < take; ++u) ops[L.nops + u] = 'I';
        L.nops += take;
        o.consumed = o.wcost = take;
        o.tcons = 0;
        o.reads = 0;
        ok = true;
    } else {
        const Planes tp = load_planes_bits(P.planes, P.plane_words, L.txt + L.t, w.n);
#ifdef GA_THREAD_STATS
        const int lane = threadIdx.x & 31;
        const long long c0 = clock64();
#endif
#if GA_COLD_COLS
        bt.jhot = w.n - GA_COLD_COLS;
#endif
#ifdef GA_CHECK
        bt.jlo = band_jstore(w.n, w.budget);
        bt.jhi = w.n;
        bt.bad = false;
#endif
        uint32_t okm = dc_band(pp, tp, w.m, w.n, band_jstore(w.n, w.budget), bt);
#ifdef GA_THREAD_STATS
        const long long c1 = clock64();
        GA_STAT(8, c1 - c0);
#endif
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
        ok = tb_band<false>(bt, pp, tp, w.m, w.n, d_min, w.budget, P.prio_lut, ops, L.nops, o);
#ifdef GA_CHECK
        if (bt.bad) ok = false;  // PrunedAccess: the pair fails as GA_STUCK
#endif
#ifdef GA_THREAD_STATS
        GA_STAT(9, clock64() - c1);
#endif
    }
    if (!ok) {
        finish(P, L, 3);
        return WIN_NEXT;
    }
    book(P, L, w, d_min, o);
    return WIN_NEXT;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    return (uint64_t)__shfl_sync(FULL, (uint32_t)(v >> 32), src) << 32 | __shfl_sync(FULL, (uint32_t)v, src);
}

// ---- lane groups: the latency path for batches far smaller than the
// resident lanes (genasm_thread_kernel<false, true>; DESIGN 3).  Each
// half-warp owns one pair; lane q of the group computes band level q (0..15)
// of every column as a wavefront -- at step s it evaluates column
// j = s - q + 1, R[q-1][j] from lane q-1 by shuffle -- so a window's DC takes
// n + 15 steps of one level each instead of n columns of 16 levels on one
// lane.  The window's band table is in shared memory, [column][level]
// unrotated (the band tier's exactness argument needs no rotation; rotating
// levels 8..15 only served the pairing of dc_band), and the group's 16 lanes
// trace back from it together (group_tb). ----
constexpr int kGroupLanes = 16;
constexpr int kGroupTabWords = 64 * thr::kFastLevels + 16;  // + 16: the two groups' banks differ

struct GroupTab {
    const uint32_t* base;  // [column - 1][level]
#ifdef GA_CHECK
    int jlo, jhi;
    mutable bool bad;
#endif
    __device__ __forceinline__ uint32_t get(int k, int c) const {
#ifdef GA_CHECK
        if (!GA_ASSERT(c >= jlo && c <= jhi && k >= 0 && k < thr::kFastLevels, 1, c, k)) {
            bad = true;
            return 0xffffffffu;
        }
#endif
        return base[(c - 1) * thr::kFastLevels + k];
    }
    __device__ __forceinline__ int wi(int e) const { return e; }
    __device__ __forceinline__ uint32_t bit(uint32_t w, int e, int b) const {
        return (w >> (b & 31)) & 1u;
    }
};

// mismatch word of column j (1..n) in the window's band coordinates
// (dc_band's two column ranges in one)
__device__ __forceinline__ uint32_t band_pm(const thr::Planes& pp, const thr::Planes& tp, int m,
                                            int n, int j) {
    const int oj = m - n - 16 + j;
    if (oj <= 0) {
        const int sh = -oj;  // virtual bits at the bottom of the band
        const uint32_t valid = sh < 32 ? ~0u << sh : 0u;
        return thr::pm_word((uint32_t)(pp.b0 << sh), (uint32_t)(pp.b1 << sh), (uint32_t)(pp.bn << sh),
                            tp, j - 1) & valid;
    }
    return thr::pm_word((uint32_t)(pp.b0 >> oj), (uint32_t)(pp.b1 >> oj), (uint32_t)(pp.bn >> oj), tp,
                        j - 1);
}

// Traceback of a group's window by its 16 lanes (backtrace.py:88-160), the
// walk of coop_tb on the group's band table: lane q evaluates the state q
// diagonal ('=') steps ahead; the first lane whose step is not '=' (ballot)
// ends the run and its step is taken, so a run of up to 16 '=' and the edit
// after it cost one round of shared-memory reads.  All 32 lanes run the
// rounds (a group without a walk, or done, idles through them); counters are
// group-uniform.  Returns false if the walk got stuck (or, GA_CHECK, read a
// column below jlo: PrunedAccess).
__device__ __forceinline__ bool group_tb(const uint32_t* gtab, bool walk, const thr::Planes& pp,
                                         const thr::Planes& tp, int m, int n, int d_min, int budget,
                                         int jlo, uint64_t prio_lut, uint8_t* ops, int64_t& nops,
                                         thr::TbOut& o, int q, int lead) {
    using namespace thr;
    constexpr uint32_t kChars = '=' | 'X' << 8 | 'I' << 16 | 'D' << 24;
    const int o0 = m - n - 16;
    bool bad = false;
    auto word = [&](int e, int c) -> uint32_t {
        if (!GA_ASSERT(c >= jlo && c <= n && e >= 0 && e < kFastLevels, 1, c, e)) {
            bad = true;
            return 0xffffffffu;
        }
        return gtab[(c - 1) * kFastLevels + e];
    };
    int d = d_min, j = n, i = m - 1;
    o.consumed = o.tcons = o.wcost = 0;
    o.reads = 0;
    unsigned racc = 0;  // this lane's share of the entry reads
    bool done = !walk, ok = true;
#ifdef GA_THREAD_STATS
    const int lane = q + lead;
    int rounds = 0;
#endif
    for (;;) {
        if (!done) {
            if (i < 0 || o.consumed >= budget) {
                done = true;
            } else if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
                if (i + 1 > d) {
                    ok = false;
                } else {
                    const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
                    for (int u = q; u < take; u += kGroupLanes) ops[nops + u] = 'I';
                    nops += take;
                    o.wcost += take;
                    o.consumed += take;
                }
                done = true;
            }
        }
        if (!__any_sync(FULL, !done)) break;
#ifdef GA_THREAD_STATS
        ++rounds;
#endif
        const int jq = j - q, iq = i - q;
        int op = 4;  // this lane's state is past a limit (or the group is done): the run stops
        unsigned rd = 0;
        const uint64_t eqv = diag_eq(pp, tp, i - j + 1);  // symbol equality along the diagonal
        if (!done && iq >= 0 && o.consumed + q < budget && jq >= 1) {
            const bool symeq = (eqv >> (jq - 1)) & 1ull;
            const int dm1 = d > 0 ? d - 1 : 0;
            const int u = i - (o0 + j);  // band position of (iq, jq): the same along the diagonal
            uint32_t mb = 0, sb = 0, db, ib = 0;
            if (jq == 1) {  // column 0 = init(m, .): bit x inactive iff x >= level
                mb = iq - 1 >= d;
                sb = iq - 1 >= d - 1;
                db = iq >= d - 1;
            } else {
                const uint32_t w1 = word(dm1, jq - 1);
                if (iq >= 1) {
                    mb = (word(d, jq - 1) >> (u & 31)) & 1u;
                    sb = (w1 >> (u & 31)) & 1u;
                }
                db = (w1 >> ((u + 1) & 31)) & 1u;
            }
            if (iq >= 1) ib = (word(dm1, jq) >> ((u - 1) & 31)) & 1u;
            const bool dpos = d > 0;
            const bool mok = symeq && (iq == 0 || !mb);
            const bool sok = dpos && (iq == 0 || !sb);
            const bool iok = dpos && (iq == 0 || !ib);
            const bool dok = dpos && !db;
            const unsigned okm =
                (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
            op = (int)((prio_lut >> (4 * okm)) & 0xFu);
            rd = (unsigned)(jq >= 2) + (dpos ? (unsigned)(jq >= 2) + 1u : 0u);
        }
        const unsigned nz = (__ballot_sync(FULL, op != OPC_M) >> lead) & 0xffffu;
        const int f = nz ? __ffs(nz) - 1 : kGroupLanes;
        const int opf = __shfl_sync(FULL, op, lead + (f & (kGroupLanes - 1)));
        if (done) continue;
        const bool taken = f < kGroupLanes && opf <= OPC_D;  // lane f's step is taken too
        racc += (q < f || (taken && q == f)) ? rd : 0u;
        j -= f;
        i -= f;
        o.consumed += f;
        o.tcons += f;
        nops += f;
        if (f == kGroupLanes || opf == 4) continue;
        if (opf > OPC_D) {
            ok = false;
            done = true;
            continue;
        }
        if (q == 0) ops[nops] = (uint8_t)(kChars >> (8 * opf));
        ++nops;
        const int mj = opf != OPC_I, mi = opf != OPC_D;
        j -= mj;
        i -= mi;
        d -= 1;
        o.consumed += mi;
        o.tcons += mj;
        o.wcost += 1;
    }
#pragma unroll
    for (int x = kGroupLanes / 2; x >= 1; x >>= 1) racc += __shfl_xor_sync(FULL, racc, x);
    o.reads = racc;
#ifdef GA_THREAD_STATS
    GA_STAT(13, rounds);
#endif
    const bool any_bad = ((__ballot_sync(FULL, bad) >> lead) & 0xffffu) != 0;
    return ok && !any_bad;
}

// One band-tier window per group (all 32 lanes call it; a group without a
// pair idles through the shared steps).  The leader's return: WIN_HARD (state
// untouched) if d_min > 15 and k allows more; otherwise the window is booked.
__device__ __forceinline__ int group_window(const KernelParams& P, Lane& L, uint32_t* gtab,
                                            uint32_t* gpm, int lane) {
    using namespace thr;
    const int q = lane & (kGroupLanes - 1);
    const int lead = lane & ~(kGroupLanes - 1);
    const int K = P.k;
#ifdef GA_THREAD_STATS
    const long long g0 = clock64();
#endif
    Win w{};
    int run = 0;  // 1: the group computes a DC this step
    if (q == 0 && L.pair >= 0) {
        w = window_of(P, L);
        run = 1;
        if (w.n == 0) {  // R[d][0] = init(m, d) solves iff d >= m (band_window)
            run = 0;
            if (w.m > K) {
                finish(P, L, 1);
            } else {
                const int take = w.m < w.budget ? w.m : w.budget;
                uint8_t* ops = P.ops + L.ops;
                for (int u = 0; u < take; ++u) ops[L.nops + u] = 'I';
                L.nops += take;
                TbOut o;
                o.consumed = o.wcost = take;
                o.tcons = 0;
                o.reads = 0;
                book(P, L, w, w.m, o);
            }
        }
    }
    run = __shfl_sync(FULL, run, lead);
    // (every lane of the warp runs each shuffle: no shuffle under a condition)
    const int m = __shfl_sync(FULL, w.m, lead);
    const int wn = __shfl_sync(FULL, w.n, lead);
    const int n = run ? wn : 0;
    const int budget = __shfl_sync(FULL, w.budget, lead);
    const int64_t pat_at = (int64_t)shfl64((uint64_t)(L.pat + w.p), lead);
    const int64_t txt_at = (int64_t)shfl64((uint64_t)(L.txt + L.t), lead);
    Planes pp{}, tp{};
    if (run) {
        pp = load_planes_bits(P.planes, P.plane_words, pat_at, m);
        tp = load_planes_bits(P.planes, P.plane_words, txt_at, n);
        for (int x = q; x < n; x += kGroupLanes) gpm[x] = band_pm(pp, tp, m, n, x + 1);
    }
    const int jstore = band_jstore(n, budget);
    __syncwarp();  // mismatch words in; the previous window's table is no longer read
#ifdef GA_THREAD_STATS
    const long long g1 = clock64();
    GA_STAT(12, g1 - g0);
#endif
    // the wavefront: lane q holds level q
    const int o0 = m - n - 16;
    uint32_t c = init_band(m, q, o0);                     // R[q][j-1]
    uint32_t a = q > 0 ? init_band(m, q - 1, o0) : 0u;    // R[q-1][j-1]
    uint32_t out = c;
    const int S = __reduce_max_sync(FULL, run ? n + kGroupLanes - 1 : 0);
    for (int s = 0; s < S; ++s) {
        const uint32_t b = __shfl_up_sync(FULL, out, 1, kGroupLanes);  // R[q-1][j]
        const int j = s - q + 1;
        const bool valid = (unsigned)(j - 1) < (unsigned)n;
        const uint32_t pm = gpm[valid ? j - 1 : 0];
        const uint32_t g = and3(orand(c, pm, a), rotr1(a), rotl1(b));
        const uint32_t nc = q == 0 ? (c | pm) : g;
        a = valid ? b : a;
        c = valid ? nc : c;
        out = c;
        if (valid && j >= jstore) gtab[(j - 1) * thr::kFastLevels + q] = c;
    }
    __syncwarp();  // the table is complete
    // levels with R[d][n] bit m-1 (band bit 15) active
    const unsigned okv = __ballot_sync(FULL, run && !((c >> 15) & 1u));
#ifdef GA_THREAD_STATS
    const long long g2 = clock64();
    GA_STAT(8, g2 - g1);
#endif
    uint32_t okm = (okv >> lead) & 0xffffu;
    const int lim = K < 15 ? K : 15;
    okm &= (2u << lim) - 1u;
    int r = WIN_NEXT;
    if (q == 0 && run && !okm) {
        if (K <= 15) finish(P, L, 1);
        else r = WIN_HARD;
    }
    // the walk, by the group's 16 lanes (group_tb); the leader books it
    const bool walk = run && okm;
    const int d_min = okm ? __ffs(okm) - 1 : 0;
    int64_t nops = (int64_t)shfl64((uint64_t)L.nops, lead);
    uint8_t* ops = P.ops + (int64_t)shfl64((uint64_t)L.ops, lead);
    TbOut o;
#ifdef GA_GROUP_SERIAL_TB
    bool ok = true;
    if (q == 0 && walk) {
        GroupTab gt{gtab};
#ifdef GA_CHECK
        gt.jlo = jstore;
        gt.jhi = n;
        gt.bad = false;
#endif
        ok = tb_band<false>(gt, pp, tp, m, n, d_min, budget, P.prio_lut, ops, nops, o);
#ifdef GA_CHECK
        if (gt.bad) ok = false;
#endif
    }
#else
    const bool ok = group_tb(gtab, walk, pp, tp, m, n, d_min, budget, jstore, P.prio_lut, ops, nops, o,
                             q, lead);
#endif
    if (q == 0 && walk) {
        L.nops = nops;
        if (ok) book(P, L, w, d_min, o);
        else finish(P, L, 3);
    }
#ifdef GA_THREAD_STATS
    GA_STAT(9, clock64() - g2);
#endif
    return r;
}

// One pass of the full tier's wavefront: lane q computes level d = d0+q of
// full-width rows (distance.py:125-149, two 32-bit words); at step s it
// evaluates column j = s - q + 1, taking R[d-1][j] from lane q-1 by shuffle
// (lane q-1 produced it the step before).  Lane 0 of a later pass (kCarry)
// reads R[d0-1][j] -- lane 31's rows of the pass before, which coop_dc copies
// to shared memory between the passes; the first pass has no carry and holds
// level 0.  Rows go to out[s * 32] (step-major, full_index).  The steps are
// branch-free: a lane outside 1 <= j <= n computes and discards.  Measured on
// the warp's own (tools/coop_bench.cu, cycles per 95-step pass, one warp per
// SM partition): a carry load in the first pass's steps, even predicated off,
// 11.5 k against 6-8 k without; the carry stored and loaded through shared
// memory inside the steps (lane 31 stores, lane 0 loads) 13.4-13.9 k; the
// next step's mismatch words loaded a step ahead 9.5 k against 8.0 k.
template <bool kCarry>
__device__ __forceinline__ void coop_pass(int m, int n, int d, uint64_t* out, const uint2* pmt,
                                          int q, uint32_t& cl, uint32_t& ch) {
    using namespace thr;
    const uint64_t a0 = d > 0 ? init_row64(m, d - 1) : 0ull;  // R[d-1][0]
    uint32_t al = (uint32_t)a0, ah = (uint32_t)(a0 >> 32);
    uint32_t ol = 0, oh = 0;  // this lane's last output
    const bool lvl0 = !kCarry && q == 0;
    const bool keep = d <= m;  // d_min <= m: no level above m is ever read
    const int S = n + kFullLevels - 1;
    // lane 0 of a later pass: R[d0-1][s+1] from the carry row coop_dc copied
    // to pmt[64 + s], read a step ahead
    uint2 cv = kCarry ? pmt[64] : make_uint2(0u, 0u);
#pragma unroll 2
    for (int s = 0; s < S; ++s) {
        uint32_t bl = __shfl_up_sync(FULL, ol, 1), bh = __shfl_up_sync(FULL, oh, 1);
        const int j = s - q + 1;
        const bool valid = (unsigned)(j - 1) < (unsigned)n;
        if (kCarry) {
            bl = q == 0 ? cv.x : bl;
            bh = q == 0 ? cv.y : bh;
            cv = pmt[64 + (s + 1 < n ? s + 1 : 0)];
        }
        const uint2 pm = pmt[valid ? j - 1 : 0];
        const uint32_t xl = cl << 1, xh = shl1_hi(cl, ch);
        uint32_t nl = and3(orand(xl, pm.x, al << 1), bl << 1, al);
        uint32_t nh = and3(orand(xh, pm.y, shl1_hi(al, ah)), shl1_hi(bl, bh), ah);
        if (!kCarry) {  // level 0: the match edge only
            nl = lvl0 ? (xl | pm.x) : nl;
            nh = lvl0 ? (xh | pm.y) : nh;
        }
        al = valid ? bl : al;
        ah = valid ? bh : ah;
        cl = valid ? nl : cl;
        ch = valid ? nh : ch;
        ol = cl;
        oh = ch;
        if (valid && keep &&
            GA_ASSERT((d >> 5) * (96 * kFullLevels) + s * kFullLevels + q < kBandWordsPerWarp / 2, 7,
                      d, j))
            out[(size_t)s * kFullLevels] = (uint64_t)nh << 32 | nl;
    }
}

// Full tier, the whole warp on one window: passes of 32 levels (coop_pass),
// rows stored to tab[full_index(d, j)], until a level <= k has R[d][n] bit
// m-1 active or the passes cover kmax.  Returns that d_min, or -1.  pmt: 128
// words of shared memory, the window's mismatch words and the carry row.
__device__ __forceinline__ int coop_dc(const thr::Planes& pp, const thr::Planes& tp, int m, int n,
                                       int K, int kmax, uint64_t* tab, uint2* pmt, int lane) {
    using namespace thr;
    const int q = lane;
    {  // the window's full-width mismatch words, one per column, in shared memory
        const uint32_t p0l = (uint32_t)pp.b0, p0h = (uint32_t)(pp.b0 >> 32);
        const uint32_t p1l = (uint32_t)pp.b1, p1h = (uint32_t)(pp.b1 >> 32);
        const uint32_t pnl = (uint32_t)pp.bn, pnh = (uint32_t)(pp.bn >> 32);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int x = q + 32 * h;  // column x+1
            const uint32_t s0 = bcast(tp.b0, x), s1 = bcast(tp.b1, x), sn = bcast(tp.bn, x);
            pmt[x] = make_uint2((p0l ^ s0) | (p1l ^ s1) | pnl | sn,
                                (p0h ^ s0) | (p1h ^ s1) | pnh | sn);
        }
        __syncwarp();
    }
    // d_min <= m (m deletions always align), so no pass goes beyond level m and
    // rows above m are never stored: the third pass of a W = 64 window holds
    // level 64 alone, inside the warp's region (rows 65..95 of that
    // pass used to overrun it)
    for (int d0 = 0; d0 <= K && d0 <= kmax && d0 <= m; d0 += kFullLevels) {
        const int d = d0 + q;
        const uint64_t c0 = init_row64(m, d);  // R[d][0]
        uint32_t cl = (uint32_t)c0, ch = (uint32_t)(c0 >> 32);
        uint64_t* out = tab + (size_t)(d0 >> 5) * (96 * kFullLevels) + q;
        if (d0 == 0) coop_pass<false>(m, n, d, out, pmt, q, cl, ch);
        else coop_pass<true>(m, n, d, out, pmt, q, cl, ch);
        __syncwarp();  // rows are read by the next pass and the traceback
        const bool hit = d <= K && d <= m && !(((uint64_t)ch << 32 | cl) >> (m - 1) & 1ull);
        const unsigned hm = __ballot_sync(FULL, hit);
        if (hm) return d0 + __ffs(hm) - 1;
        // another pass: its lane 0 needs this pass's last level, R[d0+31][j]
        // (lane 31's row of step j+30), copied once to shared memory so the
        // pass's steps read it there instead of waiting on L2 (a desynchronised
        // pair runs two passes per window)
        {
            const uint64_t* last = tab + (size_t)(d0 >> 5) * (96 * kFullLevels) + (kFullLevels - 1);
            for (int x = q; x < n; x += kFullLevels) {
                const uint64_t v = last[(size_t)(x + kFullLevels - 1) * kFullLevels];
                pmt[64 + x] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
            }
            __syncwarp();
        }
    }
    return -1;
}

// hand-over list: pairs whose windows exceed one full-tier pass; the warps
// that run out of pairs finish them (tail of genasm_thread_kernel)
struct HandList {
    int32_t* list;      // pair ids by ticket, -1 until published
    unsigned* count;    // tickets handed out to producers
    unsigned* claim;    // tickets taken by consumers
    unsigned* sm_claims;  // per SM (by %smid): fresh pairs taken / warps lingering
    unsigned* linger;
    unsigned* started;  // blocks of this launch that have started
    int sm_share;       // fresh pairs per SM when pairs are fewer than lanes (else 0)
    int linger_cap;     // warps per SM that stay to serve hand-overs (else 0)
};

// %smid numbering need not be contiguous: per-SM arrays have kSmSlots entries
constexpr int kSmSlots = 1024;
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r & (kSmSlots - 1);
}

__device__ __forceinline__ void hand_over(const KernelParams& P, Lane& L, const HandList& H) {
    PairResult* r = reinterpret_cast<PairResult*>(P.results) + L.pair;
    r->fail_window = L.widx;
    r->cost = L.cost;
    r->text_consumed = L.t;
    r->rows_computed = L.rows;
    r->ops_len = L.nops;
    r->entry_reads = L.reads;
    r->entry_writes = L.writes;
    r->words_allocated = L.words;
    const unsigned slot = atomicAdd(H.count, 1u);
    __threadfence();  // the state is visible before the id
    atomicExch(H.list + slot, L.pair);
    L.pair = -1;
}

__device__ __forceinline__ void resume_pair(const KernelParams& P, Lane& L, int pair) {
    fresh_pair(P, L, pair);
    // the parked state was written by another SM: read it from L2 (volatile),
    // never from a line this SM's L1 may hold from an earlier resume of the
    // record next to it
    const volatile PairResult* r = reinterpret_cast<const volatile PairResult*>(P.results) + pair;
    L.widx = r->fail_window;
    L.cost = r->cost;
    L.t = r->text_consumed;
    L.rows = r->rows_computed;
    L.nops = r->ops_len;
    L.reads = r->entry_reads;
    L.writes = r->entry_writes;
    L.words = r->words_allocated;
}

// Traceback of a full-tier window by the whole warp (backtrace.py:88-160):
// lane q evaluates the state q diagonal ('=') steps ahead; the first lane
// whose step is not '=' (ballot) ends the run and its step is taken, so a run
// of up to 32 '=' costs one round of table reads.  The walk is warp-uniform;
// the ops go to ops[nops..], counters to o.
__device__ __forceinline__ bool coop_tb(const uint64_t* tab, const thr::Planes& pp,
                                        const thr::Planes& tp, int m, int n, int d_min, int budget,
                                        uint64_t prio_lut, uint8_t* ops, int64_t& nops,
                                        thr::TbOut& o, int lane) {
    using namespace thr;
    constexpr uint32_t kChars = '=' | 'X' << 8 | 'I' << 16 | 'D' << 24;
    // row of level e at column c (full_index); lane q reads columns j-q-1 and
    // j-q, so its rows are the uniform ones moved back q wavefront steps
    auto row = [&](int e, int c) -> uint64_t {
        if (!GA_ASSERT(c >= 1 && c <= n && e >= 0 && e <= d_min &&
                           full_index(e, c) < kBandWordsPerWarp / 2,
                       3, e, c))
            return ~0ull;
        return tab[full_index(e, c)];
    };
    int d = d_min, j = n, i = m - 1;
    o.consumed = o.tcons = o.wcost = 0;
    unsigned racc = 0;  // this lane's share of the entry reads, summed on return
    auto done = [&](bool ok) {
        o.reads = __reduce_add_sync(FULL, racc);
        return ok;
    };
    for (;;) {
        if (i < 0 || o.consumed >= budget) return done(true);
        if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
            if (i + 1 > d) return done(false);
            const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
            for (int u = lane; u < take; u += 32) ops[nops + u] = 'I';
            nops += take;
            o.wcost += take;
            o.consumed += take;
            return done(true);
        }
        const int jq = j - lane, iq = i - lane;
        int op = 4;  // this lane's state is past a limit: the run stops here
        unsigned rd = 0;
        // symbol equality along the walk's diagonal, one mask for all lanes
        const uint64_t eqv = diag_eq(pp, tp, i - j + 1);
        if (iq >= 0 && o.consumed + lane < budget && jq >= 1) {
            const bool symeq = (eqv >> (jq - 1)) & 1ull;
            const int dm1 = d > 0 ? d - 1 : 0;
            uint32_t mb = 0, sb = 0, db, ib = 0;
            if (jq == 1) {  // column 0 = init(m, .): bit x inactive iff x >= level
                mb = iq - 1 >= d;
                sb = iq - 1 >= d - 1;
                db = iq >= d - 1;
            } else {
                const uint64_t rp = row(dm1, jq - 1);
                if (iq >= 1) {
                    mb = (uint32_t)(row(d, jq - 1) >> (iq - 1)) & 1u;
                    sb = (uint32_t)(rp >> (iq - 1)) & 1u;
                }
                db = (uint32_t)(rp >> iq) & 1u;
            }
            if (iq >= 1) ib = (uint32_t)(row(dm1, jq) >> (iq - 1)) & 1u;
            const bool dpos = d > 0;
            const bool mok = symeq && (iq == 0 || !mb);
            const bool sok = dpos && (iq == 0 || !sb);
            const bool iok = dpos && (iq == 0 || !ib);
            const bool dok = dpos && !db;
            const unsigned okm =
                (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
            op = (int)((prio_lut >> (4 * okm)) & 0xFu);
            rd = (unsigned)(jq >= 2) + (dpos ? (unsigned)(jq >= 2) + 1u : 0u);
        }
        const unsigned nz = __ballot_sync(FULL, op != OPC_M);
        const int f = nz ? __ffs(nz) - 1 : 32;
        const int opf = __shfl_sync(FULL, op, f & 31);
        const bool taken = f < 32 && opf <= OPC_D;  // lane f's step is taken too
        racc += (lane < f || (taken && lane == f)) ? rd : 0u;
        j -= f;
        i -= f;
        o.consumed += f;
        o.tcons += f;
        nops += f;
        if (f == 32 || opf == 4) continue;
        if (opf > OPC_D) return done(false);
        if (lane == 0) ops[nops] = (uint8_t)(kChars >> (8 * opf));
        ++nops;
        const int mj = opf != OPC_I, mi = opf != OPC_D;
        j -= mj;
        i -= mi;
        d -= 1;
        o.consumed += mi;
        o.tcons += mj;
        o.wcost += 1;
    }
}

// One full-tier window of the pair owned by lane `owner`, computed by the
// whole warp; the owner traces back and books it.  Levels up to kmax; returns
// true (owner's state untouched) if the window needs more.
__device__ __forceinline__ bool coop_window(const KernelParams& P, Lane& L, int owner, int lane,
                                            int kmax, uint64_t* ftab, uint2* pmt) {
    const int Lp = __shfl_sync(FULL, L.Lp, owner), Lt = __shfl_sync(FULL, L.Lt, owner);
    const int widx = __shfl_sync(FULL, L.widx, owner);
    const int64_t pat = (int64_t)shfl64((uint64_t)L.pat, owner);
    const int64_t txt = (int64_t)shfl64((uint64_t)L.txt, owner);
    const int64_t tt = (int64_t)shfl64((uint64_t)L.t, owner);
    Lane V;
    V.Lp = Lp;
    V.Lt = Lt;
    V.widx = widx;
    V.t = tt;
    const Win w = window_of(P, V);
    const thr::Planes pp = thr::load_planes_bits(P.planes, P.plane_words, pat + w.p, w.m);
    const thr::Planes tp = thr::load_planes_bits(P.planes, P.plane_words, txt + tt, w.n);
    __syncwarp();  // the band tables of this step are no longer read
    int d_min;
    if (w.n == 0) {  // R[d][0] = init(m, d) solves iff d >= m
        d_min = w.m <= P.k ? w.m : -1;
    } else {
#ifdef GA_THREAD_STATS
        const long long c0 = clock64();
#endif
        d_min = coop_dc(pp, tp, w.m, w.n, P.k, kmax, ftab, pmt, lane);
#ifdef GA_THREAD_STATS
        GA_STAT(10, clock64() - c0);
        if (kmax > kFullLevels) {
            GA_STAT(14, 1);
            GA_STAT(15, clock64() - c0);
        }
#endif
        if (d_min < 0 && P.k > kmax) return true;
    }
    if (d_min < 0) {
        if (lane == owner) finish(P, L, 1);
    } else {
        // the walk, by all lanes; the owner books it
        int64_t nops = (int64_t)shfl64((uint64_t)L.nops, owner);
        uint8_t* ops = P.ops + (int64_t)shfl64((uint64_t)L.ops, owner);
        thr::TbOut o;
#ifdef GA_THREAD_STATS
        const long long c1 = clock64();
#endif
        const bool ok = coop_tb(ftab, pp, tp, w.m, w.n, d_min, w.budget, P.prio_lut, ops, nops, o,
                                lane);
#ifdef GA_THREAD_STATS
        GA_STAT(11, clock64() - c1);
        if (kmax > kFullLevels) GA_STAT(16, clock64() - c1);
#endif
        if (lane == owner) {
#ifdef GA_THREAD_STATS
            if (L.pair < 262144) g_pair_t[2][L.pair] += 1;
#endif
            L.nops = nops;
            if (ok) book(P, L, w, d_min, o);
            else finish(P, L, 3);
        }
    }
    __syncwarp();  // the table is rewritten by the next full-tier window
    return false;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Idle for about ns nanoseconds.  __nanosleep alone returns far earlier than
// asked: a config-4 profile had the idle warps' poll loop at 40 % of all
// executed instructions (about ten polls per microsecond per warp), issue
// slots taken from the warps still aligning.
__device__ __forceinline__ void idle_ns(unsigned long long ns) {
    const unsigned long long t0 = globaltimer();
    do {
        __nanosleep(1000);
    } while (globaltimer() - t0 < ns);
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
#define GA_THREAD_MINB (512 / GA_TBLOCK)  // blocks per SM the register budget must allow
#endif

// kShare: the launch has fewer pairs than lanes and the GPU to itself -- an
// equal share of the pairs per SM, and idle warps that stay to serve the
// hand-over list.  A separate instance, so the common case's code and
// register allocation do not carry it (the shared instance measured 4 %
// slower on config 3).
template <bool kShare, bool kGroup>
__global__ void __launch_bounds__(kTBlock, GA_THREAD_MINB)
genasm_thread_kernel(const KernelParams P, uint32_t* band_base, const HandList H) {
    const int lane = threadIdx.x & 31;
    // kGroup: per warp, two group band tables and two mismatch rows (dynamic)
    extern __shared__ uint32_t s_dyn[];
    uint32_t* gtab = nullptr;
    uint32_t* gpm = nullptr;
    if (kGroup) {
        uint32_t* wb = s_dyn + (threadIdx.x >> 5) * (2 * kGroupTabWords + 128);
        gtab = wb + (lane >> 4) * kGroupTabWords;
        gpm = wb + 2 * kGroupTabWords + (lane >> 4) * 64;
    }
    if ((kShare || kGroup) && threadIdx.x == 0) atomicAdd(H.started, 1u);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t* region = band_base + gw * kBandWordsPerWarp;
    BandTab bt{reinterpret_cast<uint4*>(region), lane};
#if GA_COLD_COLS
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(bt.pol));
#endif
    uint64_t* ftab = reinterpret_cast<uint64_t*>(region);  // full tier reuses the region
    __shared__ uint2 s_pm[kWarps][128];  // full tier: mismatch words per column, carry row
    uint2* pmt = s_pm[threadIdx.x >> 5];
    const unsigned lt = lanemask_lt();
    bool exhausted = false;
    bool capped = false, uncapped = false;  // this SM's share of the pairs is taken / ignored
    unsigned long long cap_q = ~0ull, cap_t = 0;  // queue position last seen while capped, when
    Lane L;
    L.pair = -1;
    for (;;) {
        // ---- free lanes take fresh pairs from the global longest-first queue ----
        const bool want = L.pair < 0 && (!kGroup || (lane & (kGroupLanes - 1)) == 0);
        unsigned freem = __ballot_sync(FULL, want);
        if (freem && !exhausted) {
            int cnt = __popc(freem);
            unsigned long long base = 0;
            if (lane == 0) {
                if (kShare && H.sm_share && !uncapped) {  // an equal share per SM
                    const int had = (int)atomicAdd(H.sm_claims + smid(), (unsigned)cnt);
                    const int left = H.sm_share - had;
                    cnt = left < 0 ? 0 : (left < cnt ? left : cnt);
                }
                base = cnt ? atomicAdd(P.queue, (unsigned long long)cnt) : 0ull;
            }
            cnt = __shfl_sync(FULL, cnt, 0);
            base = __shfl_sync(FULL, base, 0);
            if (kShare && cnt == 0) capped = true;  // this SM's share is taken (the queue may not be)
            else if (base + cnt >= (unsigned long long)P.n_pairs) exhausted = true;
            if (want && (int)__popc(freem & lt) < cnt) {
                const uint64_t idx = base + __popc(freem & lt);
                if (idx < (uint64_t)P.n_pairs) {
                    fresh_pair(P, L, P.order ? P.order[idx] : (int)idx);
                    if (L.Lp <= 0) finish(P, L, 2);  // EmptyPattern (window.py:87-88)
                }
            }
        }
        const unsigned active = __ballot_sync(FULL, L.pair >= 0);
        if (!active) {
            if (exhausted) break;
            if (kShare && capped) {
                // The share only balances the start.  An SM that never runs a
                // block of this launch would leave its share unclaimed, so a
                // capped warp with nothing to do stops once the queue is
                // empty, and takes what is left if the queue stands still for
                // 200 us (nobody else is claiming it).
                unsigned long long q = 0, tnow = 0;
                if (lane == 0) {
                    q = *(volatile unsigned long long*)P.queue;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
                }
                q = __shfl_sync(FULL, q, 0);
                tnow = __shfl_sync(FULL, tnow, 0);
                if (q >= (unsigned long long)P.n_pairs) break;
                if (q != cap_q) {
                    cap_q = q;
                    cap_t = tnow;
                } else if (tnow - cap_t > 200000ull) {
                    uncapped = true;
                    capped = false;
                }
                idle_ns(2000);
            }
            continue;
        }

        // ---- one band-tier window per active lane ----
        GA_STAT(0, 1);
        GA_STAT(1, __popc(active));
#ifdef GA_THREAD_STATS
        const long long tw0 = clock64();
#endif
        int r = WIN_NEXT;
        if (kGroup) r = group_window(P, L, gtab, gpm, lane);
        else if (L.pair >= 0) r = band_window(P, L, bt);
        if (L.pair >= 0) {
            // a pair whose windows keep leaving the band tier (unrelated or very
            // divergent sequences) is handed over: the warps that run out of
            // pairs finish it, so it does not hold its warp back
            L.streak = r == WIN_HARD ? L.streak + 1 : 0;
            if (L.streak >= (kGroup ? kStreakGroups : kStreak)) {
                hand_over(P, L, H);
                r = WIN_NEXT;
            }
        }
        unsigned hm = __ballot_sync(FULL, r == WIN_HARD);
#ifdef GA_THREAD_STATS
        GA_STAT(4, clock64() - tw0);
        const long long th0 = clock64();
#endif
        // ---- windows beyond the band tier: the warp computes each one together;
        // a window beyond level 31 hands its pair over (below) ----
        while (hm) {
            const int owner = __ffs(hm) - 1;
            hm &= hm - 1;
            GA_STAT(2, 1);
            if (coop_window(P, L, owner, lane, kFullLevels - 1, ftab, pmt) && lane == owner)
                hand_over(P, L, H);
        }
#ifdef GA_THREAD_STATS
        GA_STAT(5, clock64() - th0);
#endif
#ifndef GA_NO_DISCARD
        if (!kGroup) {
        // the step's tables are dead once every lane has traced back: drop
        // their L2 lines without write-back, so they neither go to DRAM nor
        // crowd out the tables other warps are still reading
        __syncwarp();
#pragma unroll 4
        for (int l = lane; l < kBandWordsPerWarp * 4 / 128; l += 32)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(region) + l * 128)
                         : "memory");
        __syncwarp();
        }
#endif
    }

#ifdef GA_THREAD_STATS
    {  // spread of the warps' finishing times (global ns timer)
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        if (lane == 0) {
            atomicMin(&g_thread_stats[6], tnow);
            atomicMax(&g_thread_stats[7], tnow);
        }
    }
#endif
    // P.queue[1] counts the warps past their own pairs (P.queue[0] is the
    // fresh-pair queue): hand-overs come only from warps before this point.
    // (A count of finished pairs instead -- one atomic per pair -- measured
    // 5 ms slower on config 3.)
    if ((kShare || kGroup) && lane == 0) atomicAdd(P.queue + 1, 1ull);
    bool lingering = false;
    unsigned nap = 250;
    // ---- handed-over pairs: a warp out of pairs claims the published ones,
    // one at a time, and finishes each with all lanes, every window in the
    // full tier (up to k).  It claims only while unclaimed tickets exist and
    // then exits: every producer runs this loop after its own pairs, so no
    // ticket is left behind and nobody waits for future hand-overs. ----
    for (;;) {
        int ticket = -1;
        if (lane == 0) {
            unsigned c = *(volatile unsigned*)H.claim;
            while (c < *(volatile unsigned*)H.count) {
                const unsigned prev = atomicCAS(H.claim, c, c + 1);
                if (prev == c) {
                    ticket = (int)c;
                    break;
                }
                c = prev;
            }
        }
        ticket = __shfl_sync(FULL, ticket, 0);
        if (ticket < 0) {
            // Nothing published.  Up to linger_cap warps per SM stay (while
            // pairs remain unfinished) so a pair handed over later -- an
            // unrelated or desynchronised pair whose every window needs the
            // full tier -- is taken at once instead of when its producer's
            // other pairs are done; the rest leave the SM.
            if (!kShare && !kGroup) break;
            if (!lingering) {
                // Only while every block of the launch has started: a warp
                // that waited for hand-overs while blocks of its own grid
                // could not be scheduled (another launch holding part of the
                // GPU) could wait for warps that never run.
                int stay = 0;
                if (lane == 0 && H.linger_cap &&
                    *(volatile unsigned*)H.started >= gridDim.x)
                    stay = (int)atomicAdd(H.linger + smid(), 1u) < H.linger_cap;
                if (!__shfl_sync(FULL, stay, 0)) break;
                lingering = true;
            }
            // every warp past its own pairs: no hand-over can come any more
            unsigned long long past = 0;
            if (lane == 0) past = *(volatile unsigned long long*)(P.queue + 1);
            if (__shfl_sync(FULL, past, 0) >= (unsigned long long)gridDim.x * kWarps) break;
            idle_ns(nap);
            nap = nap < 4000 ? 2 * nap : nap;
            continue;
        }
        nap = 250;
        int pair = -1;
        for (;;) {  // the producer publishes right after taking the slot
            if (lane == 0) pair = *(volatile int32_t*)(H.list + ticket);
            pair = __shfl_sync(FULL, pair, 0);
            if (pair >= 0) break;
            __nanosleep(100);
        }
        __threadfence();
        GA_ASSERT(pair < P.n_pairs, 6, pair, ticket);
        L.pair = -1;
        if (lane == 0) resume_pair(P, L, pair);
#ifdef GA_THREAD_STATS
        if (lane == 0 && pair < 262144) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            g_pair_t[3][pair] = tnow;
        }
#endif
        while (__shfl_sync(FULL, L.pair, 0) >= 0) {
            // lane 0 owns the pair; window_of() on lane 0's state drives all lanes
#ifdef GA_THREAD_STATS
            const long long tw = clock64();
#endif
            if (coop_window(P, L, 0, lane, 1 << 30, ftab, pmt)) break;  // cannot: kmax covers k
#ifdef GA_THREAD_STATS
            GA_STAT(17, clock64() - tw);
#endif
        }
    }
}

cudaError_t launch_genasm_thread(const KernelParams& base, int num_sms, cudaStream_t stream,
                                 uint32_t** scratch, size_t* cap, LaunchShape* shape) {
    if (base.W > 64) return cudaErrorInvalidValue;
    KernelParams P = base;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, genasm_thread_kernel<false, false>, kTBlock, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const char* cap_env = getenv("GA_WARPS_PER_SM");
    // 16 warps per SM measured best on config 3 (12: 3 % slower; 20 at a
    // 96-register cap: 13 % slower)
    const int warps_cap = cap_env && atoi(cap_env) > 0 ? atoi(cap_env) : 16;
    const int bcap = warps_cap / kWarps;
    if (bcap >= 1 && per_sm > bcap) per_sm = bcap;
    // every SM equally loaded; lanes pull pairs from the global queue
    const int64_t resident = (int64_t)num_sms * per_sm * kTBlock;
    // Pairs at least as many as lanes: every warp resident, lanes refill from
    // the queue.  Fewer, with the GPU to itself (the device call, a one-chunk
    // host call): still every warp, an equal share of the pairs per SM (by
    // %smid), and the warps without pairs serve the hand-over list
    // (genasm_thread_kernel<true, false>; config 4: 106 -> 83-91 ms).  Fewer in an
    // overlapped pipeline chunk: as many lanes as pairs.
    // Pairs at most an eighth of the lanes, the GPU to itself: the lane-group
    // kernel (two pairs per warp, 16 lanes each; genasm_thread_kernel<false,
    // true>), whose shorter window latency is what bounds such a batch.
    // Measured (dev_kernel, ms): config 5 22.5 -> 9.4; config 3 first 8,000
    // pairs 8.9 -> 8.6 but 17,366 pairs 10.5 -> 14.7 (two pairs per warp
    // issue more per window than one lane each once the SMs fill up); e2e
    // pipeline chunks keep the lane-per-pair kernel (2.08 -> 2.01 M/s with
    // it).  GA_LANE_GROUPS=0/1 forces the choice.
    const size_t gsmem = (size_t)kWarps * (2 * kGroupTabWords + 128) * sizeof(uint32_t);
    const char* genv = getenv("GA_LANE_GROUPS");
    const bool group = genv ? atoi(genv) != 0 : !P.overlapped && P.n_pairs * 8 <= resident;
    int per_sm_g = per_sm;
    if (group) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_g, genasm_thread_kernel<false, true>,
                                                          kTBlock, gsmem);
        if (e != cudaSuccess) return e;
        if (per_sm_g < 1) return cudaErrorInvalidConfiguration;
        if (bcap >= 1 && per_sm_g > bcap) per_sm_g = bcap;
    }
    const int sm_share = !group && P.n_pairs < resident && !P.overlapped
                             ? (int)((P.n_pairs + num_sms - 1) / num_sms) : 0;
    const int64_t lanes = P.n_pairs < resident ? P.n_pairs : resident;
    // The equal-share launch keeps only the blocks a SM's share needs, and at
    // least two: the warps beyond the share (they serve the hand-overs) take
    // issue slots from the working ones.  Config 4 (135 pairs per SM): 8 warps
    // per SM 76.0 ms, 12 83.5, 16 85.6; config 3's 17,367-pair shard 9.96 /
    // 10.37 / 9.90 ms.  GA_SHARE_BLOCKS overrides the count.
    int per_sm_share = per_sm;
    if (sm_share) {
        const char* sb = getenv("GA_SHARE_BLOCKS");
        const int need = (sm_share + kTBlock - 1) / kTBlock;
        per_sm_share = sb && atoi(sb) > 0 ? atoi(sb) : (need > 2 ? need : 2);
        if (per_sm_share > per_sm) per_sm_share = per_sm;
    }
    int grid = sm_share ? num_sms * per_sm_share : (int)((lanes + kTBlock - 1) / kTBlock > 0
                                                         ? (lanes + kTBlock - 1) / kTBlock : 1);
    if (group) {
        // a block per SM more than the pairs need, where it fits: its warps
        // find no pair and stay to take hand-overs at once (the tail below)
        const int64_t gblocks = (P.n_pairs + 2 * kWarps - 1) / (2 * kWarps) + num_sms;
        const int64_t gmax = (int64_t)num_sms * per_sm_g;
        grid = (int)(gblocks < gmax ? gblocks : gmax);
    }
    // idle warps kept to serve hand-overs: only when this launch has the GPU
    // to itself (pipeline chunks overlap each other's launches, and a warp
    // lingering in one holds a slot the next needs: e2e 2.64 -> 2.07 M/s)
    const char* lc = getenv("GA_LINGER");
    const int linger_cap = (sm_share || group) && !P.overlapped ? (lc ? atoi(lc) : 4) : 0;
    // scratch: per-warp tables | bit-planes (one word per 64 symbols per
    // plane, plus a word of slack)
    const size_t warps = (size_t)grid * kWarps;
    const size_t band_words = (warps * kBandWordsPerWarp + 63) & ~(size_t)63;
    const int64_t pw = (P.codes_len + 63) / 64 + 1;
    const size_t plane_total = ((size_t)pw * 3 * 2 + 63) & ~(size_t)63;
    const size_t list_words = ((size_t)P.n_pairs + 63 + 64) & ~(size_t)63;
    const size_t need = band_words + plane_total + list_words + 2 * kSmSlots + 32;
    if (need > *cap || !*scratch) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *cap = 0;
        e = cudaMalloc(scratch, need * 4);
        if (e != cudaSuccess) return e;
        *cap = need;
    }
    uint32_t* band = *scratch;
    uint64_t* planes = reinterpret_cast<uint64_t*>(*scratch + band_words);
    P.planes = planes;
    P.plane_words = pw;
    {
        const int64_t blocks = (pw + 255) / 256;
        planes_kernel<<<(int)(blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8), 256, 0, stream>>>(
            P.codes, P.codes_len, planes, pw);
        if ((e = cudaGetLastError())) return e;
    }
    HandList H;
    H.list = reinterpret_cast<int32_t*>(*scratch + band_words + plane_total);
    H.count = reinterpret_cast<unsigned*>(H.list + (((size_t)P.n_pairs + 63) & ~(size_t)63));
    H.claim = H.count + 1;
    H.sm_claims = *scratch + band_words + plane_total + list_words;
    H.linger = H.sm_claims + kSmSlots;
    H.started = H.linger + kSmSlots;
    H.sm_share = sm_share;
    H.linger_cap = linger_cap;
    if ((e = cudaMemsetAsync(H.sm_claims, 0, (2 * kSmSlots + 32) * 4, stream))) return e;
    if ((e = cudaMemsetAsync(H.list, 0xff, (size_t)P.n_pairs * 4, stream))) return e;
    // the tracebacks write only the ops that are not '='
    if ((e = cudaMemsetAsync(P.ops, '=', (size_t)P.ops_capacity, stream))) return e;
    if ((e = cudaMemsetAsync(H.count, 0, 2 * sizeof(unsigned), stream))) return e;
    if (group) genasm_thread_kernel<false, true><<<grid, kTBlock, gsmem, stream>>>(P, band, H);
    else if (sm_share) genasm_thread_kernel<true, false><<<grid, kTBlock, 0, stream>>>(P, band, H);
    else genasm_thread_kernel<false, false><<<grid, kTBlock, 0, stream>>>(P, band, H);
    shape->grid = grid;
    shape->block = kTBlock;
    shape->smem_bytes = group ? (int)gsmem : 0;
    shape->group = group ? kGroupLanes : 1;
    shape->blocks_per_sm = group ? per_sm_g : (sm_share ? per_sm_share : per_sm);
    shape->overflow_words_per_group = 0;
    shape->launches = 2;
    return cudaGetLastError();
}

}  // namespace genasm

#ifdef GA_CHECK
extern "C" void ga_debug_check(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, genasm::g_check, sizeof(unsigned long long) * 4);
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(genasm::g_check, z, sizeof z);
    }
}
#endif

#ifdef GA_THREAD_STATS
extern "C" void ga_debug_thread_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, genasm::g_thread_stats, sizeof(unsigned long long) * 18);
    if (reset) {
        unsigned long long z[18] = {0, 0, 0, 0, 0, 0, ~0ull, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(genasm::g_thread_stats, z, sizeof z);
        static unsigned long long pz[4][262144];
        for (int i = 0; i < 262144; ++i) pz[0][i] = ~0ull;
        cudaMemcpyToSymbol(genasm::g_pair_t, pz, sizeof pz);
    }
}
extern "C" void ga_debug_pair_times(unsigned long long* out, int n) {
    for (int k = 0; k < 4; ++k)
        cudaMemcpyFromSymbol(out + (size_t)k * n, genasm::g_pair_t, sizeof(unsigned long long) * n,
                             sizeof(unsigned long long) * 262144 * k);
}
#endif
