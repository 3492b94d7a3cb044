// genasm_thread.cu -- lane-per-pair fused DC+TB kernel (sm_100a), W <= 64.
//
// Every lane owns one pair and walks its window chain (window.py:95-120):
// DC in 32-bit diagonal bands (16 levels, exact for d_min <= 15; see
// genasm_thread.cuh), traceback from the lane's own band table, next window.
// No shuffles or cross-lane waits on the hot loop: four 32-bit operations
// per DC entry.
//
// A window the band tier cannot solve (d_min > 15, ~3 % at 15 % divergence)
// is PARKED: the pair's state goes to its result record, its id onto a global
// ring (the hard queue), and the lane takes another pair.  Parked windows are
// computed in batches: a warp that sees >= 32 of them (or has nothing else to
// do) claims up to 32 and runs one "hard step", one window per lane, in the
// wide tier (64 diagonals, 32 levels, exact for d_min <= 31; 4 instructions
// per entry for 15 of the levels, 8 for the rest).  The rare window beyond
// level 31 is then computed by the whole warp together (the full tier: lane q
// owns level q of full-width rows, a wavefront over the columns, passes of 32
// levels).  The pair goes onto the resume ring and the next free lane picks
// it up.  So a hard window costs a lane-slot of a 32-wide batch instead of a
// whole warp's wavefront, and no lane waits for another lane's hard window.
//
// Fresh pairs come from a global longest-first queue.  When pairs are fewer
// than resident lanes, each SM gets an equal share of them (the rest of its
// warps serve the hard queue).
//
// Tables, per warp, in the context's scratch slab (one 256 KB region; the
// tiers run one after another).  Band tier: [column][word quad][lane] x 16 B
// -- each column's 16 levels are 8 paired words (genasm_thread.cuh), two
// coalesced 16-byte stores per lane.  Wide tier: [column][word quad][lane]
// x 16 B, 32 paired words per column (eight 16-byte stores).  Full tier (one
// window at a time): [pass][wavefront step][level] x 8 B (full_index).  After
// each step the warp discards the region's L2 lines: the tables are dead and
// need no write-back.
#include "genasm_device.cuh"
#include "genasm_thread.cuh"

namespace genasm {

#ifdef GA_THREAD_STATS
// dev counters: [0] band steps, [1] active lanes summed over band steps,
// [2] hard steps, [3] hard windows, [4] cycles in band steps, [5] cycles in
// hard steps, [6]/[7] first/last warp exit (ns), [8]/[9] band DC/TB cycles,
// [10] full-tier windows, [11] full-tier cycles, [12] loop iterations, [13]
// hard-ring polling/claim cycles, [14] refill cycles, [15] idle cycles, [16]
// loop cycles, [18] discard cycles, [19] away lanes summed over band steps.
// Accumulated per warp (lane 0, plain adds: no contention) and summed on the
// host; [6]/[7] are global atomics at exit.
constexpr int kStatWarps = 8192;
__device__ unsigned long long g_wstats[kStatWarps][20];
__device__ unsigned long long g_thread_stats[20];
// timeline: per 1 ms slice of the launch (globaltimer), band steps and active lanes
__device__ unsigned long long g_timeline[2][256];
__device__ unsigned long long g_t0;
__device__ unsigned long long g_pair_t[2][262144];  // per pair: first window started, finished (ns)
__device__ unsigned g_pair_cta[262144];             // per pair: the CTA that finished it
__device__ unsigned g_cta_sm[8192];                 // per CTA: its SM
// per warp in shared memory while the kernel runs (a global read-modify-write
// per counter costs an L2 round trip), flushed to g_wstats at exit
__shared__ unsigned long long s_stats[32][20];
#define GA_STAT(k, v) \
    (lane == 0 ? (void)(s_stats[threadIdx.x >> 5][k] += (unsigned long long)(v)) : (void)0)
#else
#define GA_STAT(k, v) ((void)0)
#endif

// GA_CHECK: the debug build's contract checks (tools/build_check.sh).  A
// violated check records its code and source line in g_check (first one kept,
// all counted) and, where a pair is involved, fails that pair as GA_STUCK --
// the reference raises PrunedAccess for a read of an entry it never stored
// (dptable.py:20-30, raised at :183-184) and StuckTraceback for a walk with no
// active edge (backtrace.py:30-35).  Codes: 1 band-table read outside the
// stored columns or levels (PrunedAccess), 2 the same in the wide table, 3 a
// full-tier row outside the pass computed, 4 ops beyond the pair's capacity,
// 5 window distances beyond the pair's count, 6 a ring entry that is not a
// pair, 7 a table store outside the warp's region.
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
constexpr int kDeepRun = 1 << 30;  // full-tier windows a hard step may run for one pair in a row
// per-warp region (32-bit words): the wide tier's 64 columns x 32 words x 32 lanes
constexpr int kRegionWords = 64 * 32 * 32;
constexpr int kBandWords = 64 * 8 * 32;  // the band tier's part of it
// scheduling counters one 128-byte line apart: thousands of warps poll them
// while others update them atomically, and one line would serialise all of it
constexpr int kCtrStride = 32;

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
    using Word = uint32_t;
    static constexpr int kHalf = 16;
    uint4* base;  // this warp's region: [column][word quad][lane] x 16 B
    int lane;
#if GA_COLD_COLS
    int jhot;      // columns below jhot: rarely read by the traceback
    uint64_t pol;  // L2 evict-first policy
#endif
#ifdef GA_CHECK
    int jlo, jhi;     // the columns stored this window
    mutable bool bad; // a read outside them (PrunedAccess)
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
    // the word of column c holding level e
    __device__ __forceinline__ uint32_t get(int e, int c) const {
#ifdef GA_CHECK
        if (!GA_ASSERT(c >= jlo && c <= jhi && e >= 0 && e < thr::kFastLevels, 1, c, e)) {
            bad = true;
            return 0xffffffffu;
        }
#endif
        const int k = thr::packed_word(e);
        const uint32_t* p = reinterpret_cast<const uint32_t*>(base + (size_t)(c - 1) * 64 +
                                                              (k >> 2) * 32 + lane);
        return p[k & 3];
    }
    __device__ __forceinline__ uint32_t bit(uint32_t w, int e, int b) const {
        return thr::packed_bit(w, e, b);
    }
};

// wide-tier table: [column][word quad][lane] x 16 B, 32 words (16 level
// pairs) per column, 4 KB per column per warp
struct WideTab {
    using Word = uint64_t;
    static constexpr int kHalf = 32;
    uint4* base;
    int lane;
    uint64_t pol;  // L2 evict-first: read once, soon, and not worth the band tables' room
#ifdef GA_CHECK
    int jlo, jhi;
    mutable bool bad;
#endif
    __device__ __forceinline__ void put4(int j, int q, const uint32_t* w) {
        if (!GA_ASSERT(j >= 1 && j <= 64 && q >= 0 && q < 8, 7, j, q)) return;
        st_v4_policy(base + (size_t)(j - 1) * 256 + 32 * q + lane, make_uint4(w[0], w[1], w[2], w[3]),
                     pol);
    }
    __device__ __forceinline__ uint64_t get(int e, int c) const {
#ifdef GA_CHECK
        if (!GA_ASSERT(c >= jlo && c <= jhi && e >= 0 && e < thr::kWideLevels, 2, c, e)) {
            bad = true;
            return ~0ull;
        }
#endif
        const int k = thr::wide_pair(e);  // words 2k, 2k+1: quad k/2, half k%2
        const uint2* p = reinterpret_cast<const uint2*>(base + (size_t)(c - 1) * 256 +
                                                        (k >> 1) * 32 + lane) + (k & 1);
        const uint2 v = *p;
        return (uint64_t)v.y << 32 | v.x;
    }
    __device__ __forceinline__ uint32_t bit(uint64_t w, int e, int b) const {
        return thr::wide_bit(w, e, b);
    }
};

// per-lane pair state (between windows)
struct Lane {
    int pair;  // -1: none
    int Lp, Lt, widx;
    int64_t pat, txt, ops, dst;  // offsets
    int64_t t, nops, cost, rows, reads, writes, words;
};

// Work distribution state (scratch, reset per launch): the hard and resume
// rings and the per-SM fresh-pair shares (the fresh-pair queue is P.queue).
struct Sched {
    int32_t* hard;     // ring of parked pair ids, -1 = empty slot
    int32_t* resume;   // per CTA, a ring of its pairs whose hard window is done (rcap each)
    int32_t* turn;     // per CTA, a ring of its pairs waiting their turn (time slicing)
    unsigned* rctr;    // per CTA: resume head/tail at [32 c] / [32 c + 16], turn head/tail at
                       // [32 c + 4] / [32 c + 20], fresh pairs taken (snake order) at [32 c + 8]
    unsigned rmask;    // rcap - 1
    unsigned* ctr;     // [0]/[1] hard head/tail (tickets produced/claimed), [2]/[3] resume
                       // head/tail (unused: per CTA, rctr), [4] pairs in flight: parked, in
                       // a hard step or on a resume ring (held by no lane), [5] finished pairs;
                       // entry i at ctr[i * kCtrStride]
    unsigned mask;     // ring capacity - 1
    unsigned* sm_claims;  // fresh pairs taken per SM
    int sm_share;         // fresh pairs per SM (0: unlimited)
    Lane* save;           // a lane's own state while its warp runs a hard step
    int32_t* ret;         // per pair: 1 = back from a hard step, 2 = finished there
    unsigned* linger;     // per SM: idle warps staying to serve the hard ring
    int linger_cap;       // ... at most this many per SM
    int home;             // once fresh pairs run out, a lane waits for its parked pair
    int slice;            // windows a lane runs a pair before rotating it (0: never)
    int snake;            // fresh pairs dealt to CTAs in snake order (else one global queue)
    int steal;            // free lanes take waiting pairs from other CTAs' rings
    int gturn;            // one turn ring for the launch (else one per CTA)
    int steal_gap;        // take from another CTA whose queue is longer by this much
};

// hard-ring entries: the pair id, kHome set when the pair's lane waits for it
// (it returns to that lane, not to the resume ring)
constexpr int32_t kHome = 0x40000000;

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
    L.t = L.nops = L.cost = L.rows = L.reads = L.writes = L.words = 0;
}

// a failed pair: its record and the window distances it never completed (0);
// rare, kept out of line (plain values in, so the kernel parameters stay in
// the constant bank)
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

__device__ __forceinline__ void finish(const KernelParams& P, const Sched& S, Lane& L, int status) {
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
    atomicAdd(S.ctr + 5 * kCtrStride, 1u);
#ifdef GA_THREAD_STATS
    if (L.pair < 262144) {
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        g_pair_t[1][L.pair] = tnow;
        g_pair_cta[L.pair] = blockIdx.x;
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
__device__ __forceinline__ void book(const KernelParams& P, const Sched& S, Lane& L, const Win& w,
                                     int d_min, const thr::TbOut& o) {
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
    if (w.p + o.consumed >= L.Lp) finish(P, S, L, 0);
}

// gpu-scope relaxed / release accesses (no SC fences: __threadfence() is a
// fence.sc, which serialises across the GPU and made every ring operation
// cost microseconds)
__device__ __forceinline__ unsigned ld_relaxed(const void* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(void* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(void* p, unsigned v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- rings: slot = ticket & mask, -1 = empty.  A producer takes a ticket,
// waits for its slot to be empty (never, in practice: capacity > n_pairs and a
// pair sits in at most one ring) and publishes with a release store (the
// pair's parked state before its id); a consumer claims tickets, waits for
// their ids and empties the slots.  The consumer reads the state at L2
// (ld.cg) through the id it read, so it needs no acquire fence. ----
__device__ __forceinline__ void ring_push(int32_t* ring, unsigned mask, unsigned* head, int pair) {
    const unsigned t = atomicAdd(head, 1u);
    int32_t* slot = ring + (t & mask);
    while ((int)ld_relaxed(slot) >= 0) __nanosleep(64);
    st_release(slot, (unsigned)pair);
}

__device__ __forceinline__ int ring_pop(int32_t* ring, unsigned mask, unsigned ticket) {
    int32_t* slot = ring + (ticket & mask);
    int v;
    while ((v = (int)ld_relaxed(slot)) < 0) __nanosleep(32);
    st_relaxed(slot, 0xffffffffu);
    GA_ASSERT(v >= 0, 6, v, ticket);
    return v;
}

// lane 0: claim up to `want` tickets of a ring (head = produced, tail =
// claimed); returns the count, *base the first ticket
// lane 0: claim up to `want` tickets of a ring (head = produced, tail =
// claimed), at least `least` of them; returns the count, *base the first
// ticket.  `tries` bounds the CAS attempts: on the global hard ring hundreds of
// warps can see a full batch at once, and a warp with work of its own does
// better to run its band step than to keep retrying.
__device__ __forceinline__ unsigned ring_claim(unsigned* head, unsigned* tail, unsigned want,
                                               unsigned* base, unsigned least = 1,
                                               int tries = 1 << 30) {
    unsigned t = ld_relaxed(tail);
    for (; tries > 0; --tries) {
        const int avail = (int)(ld_relaxed(head) - t);
        if (avail < (int)least || want == 0) return 0;
        const unsigned cnt = (unsigned)avail < want ? (unsigned)avail : want;
        const unsigned prev = atomicCAS(tail, t, t + cnt);
        if (prev == t) {
            *base = t;
            return cnt;
        }
        t = prev;
    }
    return 0;
}

// a pair's state between windows into its result record
__device__ __forceinline__ void save_state(const KernelParams& P, const Lane& L) {
    PairResult* r = reinterpret_cast<PairResult*>(P.results) + L.pair;
    r->fail_window = L.widx;
    r->cost = L.cost;
    r->text_consumed = L.t;
    r->rows_computed = L.rows;
    r->ops_len = L.nops;
    r->entry_reads = L.reads;
    r->entry_writes = L.writes;
    r->words_allocated = L.words;
}

// park a pair: its state into the result record, `entry` onto a ring
__device__ __forceinline__ void park(const KernelParams& P, Lane& L, int32_t* ring, unsigned mask,
                                     unsigned* head, int32_t entry) {
    save_state(P, L);
    ring_push(ring, mask, head, entry);
}

// the parked state back (L2 reads: another SM wrote it, and this SM's L1 may
// hold an older copy of the record)
__device__ __forceinline__ void resume_pair(const KernelParams& P, Lane& L, int pair) {
    GA_ASSERT(pair >= 0 && pair < P.n_pairs, 6, pair, P.n_pairs);
    fresh_pair(P, L, pair);
    const PairResult* r = reinterpret_cast<const PairResult*>(P.results) + pair;
    L.widx = __ldcg(&r->fail_window);
    L.cost = __ldcg(&r->cost);
    L.t = __ldcg(&r->text_consumed);
    L.rows = __ldcg(&r->rows_computed);
    L.nops = __ldcg(&r->ops_len);
    L.reads = __ldcg(&r->entry_reads);
    L.writes = __ldcg(&r->entry_writes);
    L.words = __ldcg(&r->words_allocated);
}

enum : int { WIN_NEXT = 0, WIN_HARD = 1 };

// One band-tier window of lane L's pair.  Returns WIN_HARD (state untouched)
// if d_min > 15 and k allows more; otherwise books the window.
__device__ __forceinline__ int band_window(const KernelParams& P, const Sched& S, Lane& L,
                                           BandTab& bt) {
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
            finish(P, S, L, 1);
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
#ifdef GA_DEV_NO_HARD  // dev: band tier alone (windows beyond it fail the pair)
            if (true) {
#else
            if (K <= 15) {
#endif
                finish(P, S, L, 1);
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
        finish(P, S, L, 3);
        return WIN_NEXT;
    }
    book(P, S, L, w, d_min, o);
    return WIN_NEXT;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
    return (uint64_t)__shfl_sync(FULL, (uint32_t)(v >> 32), src) << 32 | __shfl_sync(FULL, (uint32_t)v, src);
}

// Full tier, the whole warp on one window: lane q computes level d0+q of
// full-width rows (distance.py:125-149, two 32-bit words) as a wavefront --
// at step s it evaluates column j = s - q + 1, taking R[d-1][j] from lane
// q-1 by shuffle (lane q-1 produced it the step before; lane 0 reads the row
// lane 31 stored in the previous pass) -- and stores every row to
// tab[full_index(d, j)].  Passes of 32 levels run until a level <= k has
// R[d][n] bit m-1 active.  d_min <= m (m deletions always align), so no pass
// goes beyond level m and rows above m are never stored: the third pass of a
// W = 64 window holds level 64 alone, inside the region.  Returns d_min or -1.
__device__ __forceinline__ int coop_dc(const thr::Planes& pp, const thr::Planes& tp, int m, int n,
                                       int K, uint64_t* tab, uint2* pmt, int lane) {
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
    for (int d0 = 0; d0 <= K && d0 <= m; d0 += kFullLevels) {
        const int d = d0 + q;
        uint64_t c = init_row64(m, d);                    // R[d][j-1]
        uint64_t a = d > 0 ? init_row64(m, d - 1) : 0ull; // R[d-1][j-1]
        uint32_t ol = 0, oh = 0;                          // this lane's last output
        for (int s = 0; s < n + kFullLevels - 1; ++s) {
            uint32_t bl = __shfl_up_sync(FULL, ol, 1), bh = __shfl_up_sync(FULL, oh, 1);
            const int j = s - q + 1;
            if (j >= 1 && j <= n) {
                if (q == 0 && d0 > 0) {  // R[d0-1][j]: the previous pass's last level
                    const uint64_t v = tab[full_index(d0 - 1, j)];
                    bl = (uint32_t)v;
                    bh = (uint32_t)(v >> 32);
                }
                const uint2 pmv = pmt[j - 1];
                const uint32_t pml = pmv.x, pmh = pmv.y;
                const uint32_t cl = (uint32_t)c, ch = (uint32_t)(c >> 32);
                const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32);
                const uint32_t xl = cl << 1, xh = shl1_hi(cl, ch);
                uint32_t nl, nh;
                if (d == 0) {  // level 0: the match edge only
                    nl = xl | pml;
                    nh = xh | pmh;
                } else {
                    nl = and3(orand(xl, pml, al << 1), bl << 1, al);
                    nh = and3(orand(xh, pmh, shl1_hi(al, ah)), shl1_hi(bl, bh), ah);
                }
                a = (uint64_t)bh << 32 | bl;
                c = (uint64_t)nh << 32 | nl;
                ol = nl;
                oh = nh;
                if (d <= m && GA_ASSERT(full_index(d, j) < kRegionWords / 2, 7, d, j))
                    tab[full_index(d, j)] = c;
            }
        }
        __syncwarp();  // rows are read by the next pass's lane 0 and by the traceback
        const bool hit = d <= K && d <= m && !((c >> (m - 1)) & 1ull);
        const unsigned hm = __ballot_sync(FULL, hit);
        if (hm) return d0 + __ffs(hm) - 1;
    }
    return -1;
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
    auto bit = [&](int e, int c, int x) -> uint32_t {
        if (!GA_ASSERT(c >= 1 && c <= n && e >= 0 && e <= d_min &&
                           full_index(e, c) < kRegionWords / 2,
                       3, e, c))
            return 1u;
        return (uint32_t)(tab[full_index(e, c)] >> x) & 1u;
    };
    int d = d_min, j = n, i = m - 1;
    o.consumed = o.tcons = o.wcost = 0;
    o.reads = 0;
    for (;;) {
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
            if (i + 1 > d) return false;
            const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
            for (int u = lane; u < take; u += 32) ops[nops + u] = 'I';
            nops += take;
            o.wcost += take;
            o.consumed += take;
            return true;
        }
        const int jq = j - lane, iq = i - lane;
        int op = 4;  // this lane's state is past a limit: the run stops here
        unsigned rd = 0;
        if (iq >= 0 && o.consumed + lane < budget && jq >= 1) {
            const bool symeq = !bit64(tp.bn, jq - 1) && !bit64(pp.bn, iq) &&
                               bit64(tp.b0, jq - 1) == bit64(pp.b0, iq) &&
                               bit64(tp.b1, jq - 1) == bit64(pp.b1, iq);
            const int dm1 = d > 0 ? d - 1 : 0;
            uint32_t mb = 0, sb = 0, db, ib = 0;
            if (jq == 1) {  // column 0 = init(m, .): bit x inactive iff x >= level
                mb = iq - 1 >= d;
                sb = iq - 1 >= d - 1;
                db = iq >= d - 1;
            } else {
                if (iq >= 1) {
                    mb = bit(d, jq - 1, iq - 1);
                    sb = bit(dm1, jq - 1, iq - 1);
                }
                db = bit(dm1, jq - 1, iq);
            }
            if (iq >= 1) ib = bit(dm1, jq, iq - 1);
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

        o.reads += __reduce_add_sync(FULL, (lane < f || (taken && lane == f)) ? rd : 0u);
        j -= f;
        i -= f;
        o.consumed += f;
        o.tcons += f;
        nops += f;
        if (f == 32 || opf == 4) continue;
        if (opf > OPC_D) return false;
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

// One full-tier window of the pair held by lane `owner`, computed by the
// whole warp; the owner books it (or fails the pair).  Returns the window's
// d_min (-1: failed), the same on every lane.
__device__ __forceinline__ int coop_window(const KernelParams& P, const Sched& S, Lane& L,
                                            int owner, int lane, uint64_t* ftab, uint2* pmt) {
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
    __syncwarp();  // the tables of this step are no longer read
    // no text left: R[d][0] = init(m, d) solves iff d >= m (a pair continued
    // in this tier can reach such a window; a parked one has n >= 1)
    const int d_min = w.n == 0 ? (w.m <= P.k ? w.m : -1) : coop_dc(pp, tp, w.m, w.n, P.k, ftab, pmt, lane);
    if (d_min < 0) {
        if (lane == owner) finish(P, S, L, 1);
    } else {
        // the walk, by all lanes; the owner books it
        int64_t nops = (int64_t)shfl64((uint64_t)L.nops, owner);
        uint8_t* ops = P.ops + (int64_t)shfl64((uint64_t)L.ops, owner);
        thr::TbOut o;
        const bool ok = coop_tb(ftab, pp, tp, w.m, w.n, d_min, w.budget, P.prio_lut, ops, nops, o,
                                lane);
        if (lane == owner) {
            L.nops = nops;
            if (ok) book(P, S, L, w, d_min, o);
            else finish(P, S, L, 3);
        }
    }
    __syncwarp();  // the table is rewritten by the next full-tier window
    return d_min;
}

// One hard step: the `cnt` parked windows at hard-ring tickets base.., one
// per lane, in the wide tier; windows beyond level 31 by the whole warp in the
// full tier; the pairs onto the resume ring (or finished).
// The launch's parameters in global memory, for hard_step: it is a separate
// (non-inlined) function so the band path keeps its own compact code and
// register allocation, and it reads the parameters from here so the kernel's
// own parameters stay in the constant bank (passing them by reference would
// copy them to local memory for the whole kernel).
struct HardCtx {
    KernelParams P;
    Sched S;
};

__device__ __noinline__ void hard_step(const HardCtx* __restrict__ H, uint32_t* region, uint2* pmt,
                                       int lane, unsigned cnt, unsigned base) {
    using namespace thr;
    const KernelParams& P = H->P;
    const Sched& S = H->S;
    int pair = -1;
    bool home = false;
    if ((unsigned)lane < cnt) {
        const int entry = ring_pop(S.hard, S.mask, base + lane);
        home = (entry & kHome) != 0;
        pair = entry & ~kHome;
    }
    // a ring-mode pair goes back to the CTA that parked it (its record's
    // status word holds the CTA while the pair is parked)
    const int cta = pair >= 0 && !home
                        ? __ldcg(&(reinterpret_cast<const PairResult*>(P.results) + pair)->status)
                        : 0;
    GA_ASSERT(cta >= 0 && cta < (int)gridDim.x, 6, pair, cta);
    Lane V;
    V.pair = -1;
    const int K = P.k;
    bool deep = false;  // beyond the wide tier: the full tier, by the warp
    if (pair >= 0) {
        // the window's geometry only: the rest of the parked state is read
        // after the DC, so it does not occupy registers during it
        const PairResult* rec = reinterpret_cast<const PairResult*>(P.results) + pair;
        Lane G;
        G.Lp = P.pat_len[pair];
        G.Lt = P.txt_len[pair];
        G.widx = __ldcg(&rec->fail_window);
        G.t = __ldcg(&rec->text_consumed);
        const Win w = window_of(P, G);  // n >= 1: windows without text never park
        const int64_t ppos = P.pat_off[pair] + w.p, tpos = P.txt_off[pair] + G.t;
        WideTab wt;
        wt.base = reinterpret_cast<uint4*>(region);
        wt.lane = lane;
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(wt.pol));
#ifdef GA_CHECK
        wt.jlo = wide_jstore(w.n, w.budget);
        wt.jhi = w.n;
        wt.bad = false;
#endif
        uint32_t okm;
        {
            const Planes pp = load_planes_bits(P.planes, P.plane_words, ppos, w.m);
            const Planes tp = load_planes_bits(P.planes, P.plane_words, tpos, w.n);
            okm = dc_wide(pp, tp, w.m, w.n, wide_jstore(w.n, w.budget), wt);
        }
        okm &= K < 31 ? (2u << K) - 1u : ~0u;
        resume_pair(P, V, pair);
        if (okm) {
            const int d_min = __ffs(okm) - 1;
            const Planes pp = load_planes_bits(P.planes, P.plane_words, ppos, w.m);
            const Planes tp = load_planes_bits(P.planes, P.plane_words, tpos, w.n);
            TbOut o;
#ifdef GA_DEV_NO_WTB
            o.consumed = o.tcons = o.wcost = 1; o.reads = 0;
            if (d_min < 100)
#else
            bool ok = tb_band<false, 4>(wt, pp, tp, w.m, w.n, d_min, w.budget, P.prio_lut,
                                        P.ops + V.ops, V.nops, o);
#ifdef GA_CHECK
            if (wt.bad) ok = false;
#endif
            if (ok)
#endif
                book(P, S, V, w, d_min, o);
            else
                finish(P, S, V, 3);
        } else if (K <= 31) {
            finish(P, S, V, 1);
        } else {
            deep = true;
        }
    }
    // the pairs done here go back first: the deep windows below may take a while
    auto send_back = [&](bool mine) {
        if (!mine) return;
        if (home) {  // back to the lane waiting for it
            if (V.pair >= 0) save_state(P, V);
            st_release(S.ret + pair, V.pair >= 0 ? 1u : 2u);
        } else if (V.pair >= 0) {
            park(P, V, S.resume + (size_t)cta * (S.rmask + 1), S.rmask, S.rctr + 32 * cta, V.pair);
        }
    };
    send_back(pair >= 0 && !deep);
    unsigned dm = __ballot_sync(FULL, deep);
    GA_STAT(10, __popc(dm));
#ifdef GA_THREAD_STATS
    const long long c0 = clock64();
#endif
    while (dm) {
        const int owner = __ffs(dm) - 1;
        dm &= dm - 1;
        // a window this deep usually means the pair has lost its diagonal
        // (unrelated or desynchronised sequences): its next windows are deep
        // too, so the warp keeps the pair while they stay at d_min >= 24
        // (up to kDeepRun windows) instead of sending each one round the rings
        for (int r = 0; r < kDeepRun; ++r) {
            const int dmin = coop_window(P, S, V, owner, lane, reinterpret_cast<uint64_t*>(region), pmt);
            if (dmin < 24 || __shfl_sync(FULL, V.pair, owner) < 0) break;
            GA_STAT(10, 1);
        }
    }
#ifdef GA_THREAD_STATS
    GA_STAT(11, clock64() - c0);
#endif
    send_back(deep);
    const unsigned done = __ballot_sync(FULL, (unsigned)lane < cnt && !home && V.pair < 0);
    if (lane == 0 && done) atomicSub(S.ctr + 4 * kCtrStride, (unsigned)__popc(done));
#ifndef GA_NO_DISCARD
    __syncwarp();
#pragma unroll 4
    for (int l = lane; l < kRegionWords * 4 / 128; l += 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(region) + l * 128)
                     : "memory");
    __syncwarp();
#endif
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// %smid numbering need not be contiguous: per-SM arrays have kSmSlots
// entries, indexed by %smid (bounded by %nsmid, far below this)
constexpr int kSmSlots = 1024;
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

}  // namespace

// codes -> three bit-planes: thread t packs symbols [64t, 64t+64) of each
// plane into one 64-bit word (bit 0 of the code, bit 1, code 4)
__global__ void __launch_bounds__(256) planes_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                     uint64_t* __restrict__ pl, int64_t words,
                                                     HardCtx* ctx, const KernelParams P, const Sched S) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the alignment kernel's parameters, for hard_step
        ctx->P = P;
        ctx->S = S;
    }
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

__global__ void __launch_bounds__(kTBlock, GA_THREAD_MINB)
genasm_thread_kernel(const KernelParams P, uint32_t* region_base, const Sched S,
                     const HardCtx* __restrict__ H) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t* region = region_base + gw * kRegionWords;
    BandTab bt{reinterpret_cast<uint4*>(region), lane};
#if GA_COLD_COLS
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(bt.pol));
#endif
    __shared__ uint2 s_pm[kWarps][64];  // full tier: mismatch words per column
    uint2* pmt = s_pm[threadIdx.x >> 5];
#ifdef GA_THREAD_STATS
    if (lane < 20) s_stats[threadIdx.x >> 5][lane] = 0;
    __syncwarp();
#endif
#ifdef GA_THREAD_STATS
    if (threadIdx.x == 0) g_cta_sm[blockIdx.x % 8192] = smid();
#endif
    const unsigned lt = lanemask_lt();
    const unsigned sm = (S.sm_share || S.linger_cap) ? smid() & (kSmSlots - 1) : 0u;
    unsigned* my_rctr = S.rctr + 32 * blockIdx.x;  // this CTA's resume ring
    int32_t* my_ring = S.resume + (size_t)blockIdx.x * (S.rmask + 1);
    // the turn ring (pairs waiting their time slice): one for the whole launch,
    // so every SM serves every pair and none falls behind with a slow SM; the
    // whole warp rotates at once, so its counters see one claim per warp per
    // slice
    unsigned* my_tctr = S.gturn ? S.ctr + 6 * kCtrStride : my_rctr + 4;
    int32_t* my_turn = S.gturn ? S.turn : S.turn + (size_t)blockIdx.x * (S.rmask + 1);
    const unsigned tmask = S.gturn ? S.mask : S.rmask;
    bool exhausted = false;  // the fresh-pair queue is empty (for this warp)
    bool lingering = false;  // an idle warp kept to serve the hard ring
    unsigned nap = 256;      // idle back-off (ns), doubled up to 8 us while nothing turns up
    Lane L;
    L.pair = -1;
    bool away = false;  // L.pair is parked in the hard ring and comes back to this lane
    int slice = 0;      // windows since the lane took its pair (time slicing)
    int wslice = 0;     // band steps since the warp last rotated its pairs
    unsigned steal_seed = blockIdx.x * 2654435761u + (threadIdx.x >> 5);
#ifdef GA_THREAD_STATS
    long long tloop = clock64();
#endif
    for (;;) {
        GA_STAT(12, 1);
#ifdef GA_THREAD_STATS
        const long long tr0 = clock64();
        GA_STAT(16, tr0 - tloop);  // the whole previous iteration
        tloop = tr0;
#endif
        if (away) {  // has the hard step sent the pair back?
            const unsigned f = ld_relaxed(S.ret + L.pair);
            if (f) {
                st_relaxed(S.ret + L.pair, 0u);
                if (f == 2) L.pair = -1;  // finished (or failed) in the hard step
                else resume_pair(P, L, L.pair);
                away = false;
            }
        }
        // ---- free lanes: fresh pairs while any remain (so every pair starts
        // early), then the pairs waiting on this CTA's ring ----
        unsigned freem = __ballot_sync(FULL, L.pair < 0);
        if (freem && !exhausted) {
            int want = __popc(freem);
            const unsigned rank = __popc(freem & lt);
            int64_t idx = -1;
            if (S.snake) {
                // pairs dealt to CTAs in snake order (0..C-1, C-1..0, ...) of the
                // longest-first order: every CTA gets an equal share of the
                // work whatever order the lanes ask in
                unsigned k0 = 0;
                if (lane == 0) k0 = atomicAdd(my_rctr + 8, (unsigned)want);
                k0 = __shfl_sync(FULL, k0, 0);
                const int64_t C = gridDim.x, k = (int64_t)k0 + rank;
                const int64_t r = k * C + ((k & 1) ? C - 1 - blockIdx.x : blockIdx.x);
                if (L.pair < 0) idx = r < P.n_pairs ? r : -2;
                // the CTA's last pair: exhausted once a claim reaches past it
                const int64_t kl = (int64_t)k0 + want - 1;
                const int64_t rl = kl * C + ((kl & 1) ? C - 1 - blockIdx.x : blockIdx.x);
                if (rl >= P.n_pairs) exhausted = true;
            } else {
                unsigned long long base = 0;
                if (lane == 0) {
                    if (S.sm_share) {  // this SM's share of the fresh pairs
                        const int had = (int)atomicAdd(S.sm_claims + sm, (unsigned)want);
                        const int left = S.sm_share - had;
                        want = left < 0 ? 0 : (left < want ? left : want);
                    }
                    base = want ? atomicAdd(P.queue, (unsigned long long)want) : 0ull;
                }
                want = __shfl_sync(FULL, want, 0);
                base = __shfl_sync(FULL, base, 0);
                if (want == 0 || base + want >= (unsigned long long)P.n_pairs) exhausted = true;
                if (L.pair < 0 && (int)rank < want && base + rank < (uint64_t)P.n_pairs)
                    idx = (int64_t)(base + rank);
            }
            if (idx >= 0) {
                fresh_pair(P, L, P.order ? P.order[idx] : (int)idx);
                slice = 0;
                if (L.Lp <= 0) finish(P, S, L, 2);  // EmptyPattern (window.py:87-88)
            }
            freem = __ballot_sync(FULL, L.pair < 0);
        }
        if (freem) {
            unsigned rb = 0, rc = 0;
            if (lane == 0) {
                rc = ring_claim(my_rctr, my_rctr + 16, __popc(freem), &rb);
                if (rc) atomicSub(S.ctr + 4 * kCtrStride, rc);  // held by this warp's lanes from here
            }
            rc = __shfl_sync(FULL, rc, 0);
            if (rc) {
                rb = __shfl_sync(FULL, rb, 0);
                const unsigned rank = __popc(freem & lt);
                if (L.pair < 0 && rank < rc) {
                    resume_pair(P, L, ring_pop(my_ring, S.rmask, rb + rank));
                    slice = 0;
                }
                freem = __ballot_sync(FULL, L.pair < 0);
            }
        }
        // then the pairs waiting their turn (time slicing): pairs back from a
        // hard step go first, they lost time on the trip
        if (freem) {
            unsigned rb = 0, rc = 0, src = blockIdx.x;
            if (lane == 0) {
                unsigned* tc = my_tctr;
                if (S.steal && !S.gturn && exhausted && __popc(freem) >= 16) {
                    // Balance as we go: a CTA whose queue of waiting pairs is much
                    // shorter than a random other CTA's takes from that one.  CTAs
                    // run at different speeds (SMs differ, hard steps land
                    // unevenly), and without this the slow ones finish last.
                    steal_seed = steal_seed * 1664525u + 1013904223u;
                    const unsigned vic = (blockIdx.x + 1 + (steal_seed >> 8) %
                                          (gridDim.x > 1 ? gridDim.x - 1 : 1)) % gridDim.x;
                    unsigned* vc = S.rctr + 32 * vic + 4;
                    const int mine = (int)(ld_relaxed(my_tctr) - ld_relaxed(my_tctr + 16));
                    const int theirs = (int)(ld_relaxed(vc) - ld_relaxed(vc + 16));
                    if (theirs > mine + S.steal_gap) {
                        tc = vc;
                        src = vic;
                    }
                }
                rc = ring_claim(tc, tc + (S.gturn ? kCtrStride : 16), __popc(freem), &rb);
                if (rc) atomicSub(S.ctr + 4 * kCtrStride, rc);
            }
            rc = __shfl_sync(FULL, rc, 0);
            if (rc) {
                rb = __shfl_sync(FULL, rb, 0);
                src = __shfl_sync(FULL, src, 0);
                const unsigned rank = __popc(freem & lt);
                if (L.pair < 0 && rank < rc) {
                    int32_t* tr = src == blockIdx.x ? my_turn : S.turn + (size_t)src * (S.rmask + 1);
                    resume_pair(P, L, ring_pop(tr, tmask, rb + rank));
                    slice = 0;
                }
                freem = __ballot_sync(FULL, L.pair < 0);
            }
        }
        // Still free lanes and nothing fresh: take waiting pairs from another
        // CTA's ring.  CTAs drift apart (hard steps stall the warps that run
        // them), and without stealing the ones left behind finish alone.
        if (freem && exhausted && S.steal && !S.gturn) {
            unsigned rb = 0, rc = 0, vic = 0;
            if (lane == 0) {
                steal_seed = steal_seed * 1664525u + 1013904223u;
                vic = (blockIdx.x + 1 + (steal_seed >> 8) % (gridDim.x - 1 ? gridDim.x - 1 : 1)) % gridDim.x;
                unsigned* vc = S.rctr + 32 * vic + 4;  // its turn ring
                rc = ring_claim(vc, vc + 16, __popc(freem), &rb, 1, 1);
                if (rc) atomicSub(S.ctr + 4 * kCtrStride, rc);
            }
            rc = __shfl_sync(FULL, rc, 0);
            if (rc) {
                rb = __shfl_sync(FULL, rb, 0);
                vic = __shfl_sync(FULL, vic, 0);
                const unsigned rank = __popc(freem & lt);
                if (L.pair < 0 && rank < rc) {
                    resume_pair(P, L, ring_pop(S.turn + (size_t)vic * (S.rmask + 1), S.rmask, rb + rank));
                    slice = 0;
                }
            }
        }
        const unsigned runnable = __ballot_sync(FULL, L.pair >= 0 && !away);
#ifdef GA_THREAD_STATS
        GA_STAT(14, clock64() - tr0);
#endif

        // ---- a hard step when a batch is ready, or when there is nothing else ----
#ifdef GA_THREAD_STATS
        const long long tc0 = clock64();
#endif
        int hc = 0;
        if (lane == 0) hc = (int)(ld_relaxed(S.ctr) - ld_relaxed(S.ctr + 1 * kCtrStride));
        hc = __shfl_sync(FULL, hc, 0);
#ifndef GA_DEV_NO_HARD
        if (hc >= 32 || (hc > 0 && !runnable)) {
            unsigned hb = 0, cnt = 0;
            if (lane == 0) cnt = ring_claim(S.ctr, S.ctr + 1 * kCtrStride, 32u, &hb, runnable ? 32u : 1u, 1);
            cnt = __shfl_sync(FULL, cnt, 0);
            if (cnt) {
                hb = __shfl_sync(FULL, hb, 0);
                GA_STAT(2, 1);
                GA_STAT(3, cnt);
#ifdef GA_THREAD_STATS
                const long long th0 = clock64();
#endif
                // the warp's own pairs go to the back of its CTA's ring first, so
                // other lanes move them on while this warp runs the hard step
                // (a lane waiting on its own parked pair keeps waiting)
                const bool mine = L.pair >= 0 && !away;
                const unsigned om = __ballot_sync(FULL, mine);
                if (om) {
                    if (lane == 0) atomicAdd(S.ctr + 4 * kCtrStride, (unsigned)__popc(om));  // first
                    __syncwarp();
                    if (mine) {
                        reinterpret_cast<PairResult*>(P.results)[L.pair].status = (int)blockIdx.x;
                        park(P, L, my_turn, tmask, my_tctr, L.pair);
                        L.pair = -1;
                    }
                }
                hard_step(H, region, pmt, lane, cnt, hb);
                nap = 256;
#ifdef GA_THREAD_STATS
                GA_STAT(5, clock64() - th0);
#endif
                continue;
            }
        }
#endif
#ifdef GA_THREAD_STATS
        GA_STAT(13, clock64() - tc0);  // hard-ring polling and claim attempts
#endif
        if (!runnable) {
            // Nothing to run.  A warp holding parked pairs waits for them.  An
            // empty warp exits once no pair is in flight (every unfinished pair
            // is then held by a lane of a live warp, which finishes it), so idle
            // warps leave the SMs to the next launch -- except up to linger_cap
            // per SM, which stay to serve the hard ring until every pair is done.
            const bool held = __ballot_sync(FULL, L.pair >= 0) != 0;
            if (!held && exhausted) {
                unsigned fl = 0, left = 0;
                if (lane == 0) {
                    fl = ld_relaxed(S.ctr + 4 * kCtrStride);
                    left = ld_relaxed(S.ctr + 5 * kCtrStride);  // finished pairs
                }
                fl = __shfl_sync(FULL, fl, 0);
                left = __shfl_sync(FULL, left, 0);
                if (left == (unsigned)P.n_pairs) break;  // every pair finished
                if (fl == 0 && hc <= 0 && !lingering) {
                    int stay = 0;
                    if (lane == 0 && S.linger_cap)
                        stay = (int)atomicAdd(S.linger + sm, 1u) < S.linger_cap;
                    if (!__shfl_sync(FULL, stay, 0)) break;
                    lingering = true;
                }
            }
#ifdef GA_THREAD_STATS
            const long long ti0 = clock64();
#endif
            __nanosleep(nap);
            nap = nap < 8192 ? 2 * nap : nap;
#ifdef GA_THREAD_STATS
            GA_STAT(15, clock64() - ti0);
#endif
            continue;
        }

        // ---- one band-tier window per runnable lane.  A window beyond the band
        // tier parks its pair on the hard ring: while fresh pairs remain the
        // lane takes one and the pair comes back through the resume ring; after
        // that the lane waits for its own pair (pairs stay where they are, so
        // warps do not thin out and SMs stay evenly loaded) ----
        nap = 256;
        GA_STAT(0, 1);
        GA_STAT(1, __popc(runnable));
#ifdef GA_TIMELINE
        if (lane == 0) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            atomicMin(&g_t0, tnow);
            const unsigned long long sl = (tnow - g_t0) / 1000000ull;
            if (sl < 256) {
                atomicAdd(&g_timeline[0][sl], 1ull);
                atomicAdd(&g_timeline[1][sl], (unsigned long long)__popc(runnable));
            }
        }
#endif
#ifdef GA_THREAD_STATS
        const unsigned awaym = __ballot_sync(FULL, away);  // every lane: not inside GA_STAT
        GA_STAT(19, __popc(awaym));
#endif
#ifdef GA_THREAD_STATS
        const long long tw0 = clock64();
#endif
        const bool hard = L.pair >= 0 && !away && band_window(P, S, L, bt) == WIN_HARD;
        // Time slicing: after S.slice windows a pair goes to the back of its
        // CTA's ring and the lane takes the next one.  Every pair then moves at
        // the same pace and they all finish together, instead of the ones
        // started last running on alone in a thinning tail.
        // the whole warp rotates at once (one refill's latency per slice, not
        // one per lane per step)
        wslice = wslice + 1;
        const bool rotate = S.slice && wslice >= S.slice && !hard && L.pair >= 0 && !away;
        if (wslice >= S.slice) wslice = 0;
        const unsigned rm = __ballot_sync(FULL, rotate);
        if (rm) {
            if (lane == 0) atomicAdd(S.ctr + 4 * kCtrStride, (unsigned)__popc(rm));  // first
            __syncwarp();
            if (rotate) {
                reinterpret_cast<PairResult*>(P.results)[L.pair].status = (int)blockIdx.x;
                park(P, L, my_turn, tmask, my_tctr, L.pair);
                L.pair = -1;
            }
        }
        const unsigned hm = __ballot_sync(FULL, hard);
        if (hm) {
            if (!exhausted || !S.home) {
                if (lane == 0) atomicAdd(S.ctr + 4 * kCtrStride, (unsigned)__popc(hm));  // first
                __syncwarp();
                if (hard) {
                    reinterpret_cast<PairResult*>(P.results)[L.pair].status = (int)blockIdx.x;
                    park(P, L, S.hard, S.mask, S.ctr, L.pair);
                    L.pair = -1;
                }
            } else if (hard) {
                park(P, L, S.hard, S.mask, S.ctr, L.pair | kHome);
                away = true;
            }
        }
#ifdef GA_THREAD_STATS
        GA_STAT(4, clock64() - tw0);
#endif
#ifdef GA_THREAD_STATS
        const long long td0 = clock64();
#endif
#ifndef GA_NO_DISCARD
        // the step's tables are dead once every lane has traced back: drop
        // their L2 lines without write-back, so they neither go to DRAM nor
        // crowd out the tables other warps are still reading
        __syncwarp();
#pragma unroll 4
        for (int l = lane; l < kBandWords * 4 / 128; l += 32)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(region) + l * 128)
                         : "memory");
        __syncwarp();
#endif
#ifdef GA_THREAD_STATS
        GA_STAT(18, clock64() - td0);
#endif
    }

#ifdef GA_THREAD_STATS
    {  // spread of the warps' finishing times (global ns timer)
        unsigned long long tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        GA_STAT(17, clock64() - tloop);
        __syncwarp();
        if (lane < 20) g_wstats[gw % kStatWarps][lane] += s_stats[threadIdx.x >> 5][lane];
        if (lane == 0) {
            atomicMin(&g_thread_stats[6], tnow);
            atomicMax(&g_thread_stats[7], tnow);
        }
    }
#endif
}

// ring capacity: a power of two above the pair count
static unsigned ring_capacity(int64_t n) {
    unsigned c = 64;
    while ((int64_t)c < n + 64) c <<= 1;
    return c;
}

cudaError_t launch_genasm_thread(const KernelParams& base, int num_sms, cudaStream_t stream,
                                 uint32_t** scratch, size_t* cap, LaunchShape* shape) {
    if (base.W > 64) return cudaErrorInvalidValue;
    KernelParams P = base;
    int per_sm = 0;
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, genasm_thread_kernel, kTBlock, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const char* cap_env = getenv("GA_WARPS_PER_SM");
    // 16 warps per SM measured best on config 3 (12: 3 % slower; 20 at a
    // 96-register cap: 13 % slower)
    const int warps_cap = cap_env && atoi(cap_env) > 0 ? atoi(cap_env) : 16;
    const int bcap = warps_cap / kWarps;
    if (bcap >= 1 && per_sm > bcap) per_sm = bcap;
    // persistent: every SM equally loaded, every warp resident; lanes pull
    // pairs from the global queue, warps without pairs serve the hard ring
    const int64_t resident = (int64_t)num_sms * per_sm * kTBlock;
    int grid = num_sms * per_sm;
    Sched S{};
    // pairs fewer than lanes: an equal share per SM (by %smid), so no SM runs
    // twice the chains of another
    S.sm_share = P.n_pairs < resident ? (int)((P.n_pairs + num_sms - 1) / num_sms) : 0;
    if (const char* v = getenv("GA_SM_SHARE")) S.sm_share = atoi(v) < 0 ? 0 : S.sm_share;
    // pairs at least as many as lanes: deal them to CTAs in snake order, so no
    // CTA is left with the chains others finished (first come, first served
    // gave some CTAs twice the pairs of others)
    S.snake = P.n_pairs >= resident;
    if (const char* v = getenv("GA_SNAKE")) S.snake = atoi(v) && P.n_pairs >= resident;
    const unsigned ring = ring_capacity(P.n_pairs);
    S.mask = ring - 1;
    // per-CTA resume rings: a CTA's parked pairs come back to it, so only its
    // own 4 warps contend for a ring; 4096 is far above what one CTA's 128
    // lanes can have parked and returned at once
    const unsigned rcap = ring_capacity(P.n_pairs < 4032 ? P.n_pairs : 4032);
    S.rmask = rcap - 1;
    // scratch (32-bit words): per-warp regions | bit-planes (one word per 64
    // symbols per plane, plus a word of slack) | 2 rings | counters | per-SM
    // claims | saved lane states
    const size_t warps = (size_t)grid * kWarps;
    auto up = [](size_t x) { return (x + 63) & ~(size_t)63; };
    const size_t region_words = up(warps * kRegionWords);
    const int64_t pw = (P.codes_len + 63) / 64 + 1;
    const size_t plane_total = up((size_t)pw * 3 * 2);
    const size_t ring_words = up(2 * (size_t)ring + 2 * (size_t)grid * rcap);
    const size_t rctr_words = up((size_t)grid * 32);
    const size_t ctr_words = 8 * kCtrStride;
    const size_t sm_words = kSmSlots;
    const size_t save_words = up(warps * 32 * sizeof(Lane) / 4);
    const size_t ret_words = up((size_t)P.n_pairs + 1);
    const size_t ctx_words = up((sizeof(HardCtx) + 3) / 4);
    const size_t need = region_words + plane_total + ring_words + ctr_words + 2 * sm_words +
                        rctr_words + save_words + ret_words + ctx_words;
    if (need > *cap || !*scratch) {
        if (*scratch) cudaFree(*scratch);
        *scratch = nullptr;
        *cap = 0;
        e = cudaMalloc(scratch, need * 4);
        if (e != cudaSuccess) return e;
        *cap = need;
    }
    uint32_t* w = *scratch;
    uint32_t* regions = w;
    w += region_words;
    uint64_t* planes = reinterpret_cast<uint64_t*>(w);
    w += plane_total;
    S.hard = reinterpret_cast<int32_t*>(w);
    S.resume = S.hard + ring;
    S.gturn = getenv("GA_GTURN") ? atoi(getenv("GA_GTURN")) : 0;
    S.steal_gap = getenv("GA_STEAL_GAP") ? atoi(getenv("GA_STEAL_GAP")) : 48;
    S.turn = S.resume + (size_t)grid * rcap;  // per-CTA turn rings, or the first `ring` words
    w += ring_words;
    S.ctr = w;
    w += ctr_words;
    S.sm_claims = w;
    w += sm_words;
    S.linger = w;
    w += sm_words;
    S.rctr = w;
    w += rctr_words;
    S.save = reinterpret_cast<Lane*>(w);
    w += save_words;
    S.ret = reinterpret_cast<int32_t*>(w);
    w += ret_words;
    HardCtx* hctx = reinterpret_cast<HardCtx*>(w);
    S.linger_cap = getenv("GA_LINGER") ? atoi(getenv("GA_LINGER")) : 0;
    S.home = getenv("GA_HOME") ? atoi(getenv("GA_HOME")) : 0;
    S.slice = getenv("GA_SLICE") ? atoi(getenv("GA_SLICE")) : 16;
    S.steal = getenv("GA_STEAL") ? atoi(getenv("GA_STEAL")) : 1;
    P.planes = planes;
    P.plane_words = pw;
    {
        const int64_t blocks = (pw + 255) / 256;
        planes_kernel<<<(int)(blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8), 256, 0, stream>>>(
            P.codes, P.codes_len, planes, pw, hctx, P, S);
        if ((e = cudaGetLastError())) return e;
    }
    if ((e = cudaMemsetAsync(S.hard, 0xff, (2 * (size_t)ring + 2 * (size_t)grid * rcap) * 4, stream))) return e;
    // ring counters, per-SM claims and lingerers, per-CTA resume counters
    // (adjacent) to 0; no pair returned
    if ((e = cudaMemsetAsync(S.ctr, 0, (ctr_words + 2 * sm_words + rctr_words) * 4, stream))) return e;
    if ((e = cudaMemsetAsync(S.ret, 0, (size_t)P.n_pairs * 4, stream))) return e;
    // the tracebacks write only the ops that are not '='
    if ((e = cudaMemsetAsync(P.ops, '=', (size_t)P.ops_capacity, stream))) return e;
    genasm_thread_kernel<<<grid, kTBlock, 0, stream>>>(P, regions, S, hctx);
    shape->grid = grid;
    shape->block = kTBlock;
    shape->smem_bytes = 0;
    shape->group = 1;
    shape->blocks_per_sm = per_sm;
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
extern "C" void ga_debug_pair_times(unsigned long long* out, int n) {
    cudaMemcpyFromSymbol(out, genasm::g_pair_t, sizeof(unsigned long long) * n, 0);
    cudaMemcpyFromSymbol(out + n, genasm::g_pair_t, sizeof(unsigned long long) * n,
                         sizeof(unsigned long long) * 262144);
    static unsigned c[262144];
    cudaMemcpyFromSymbol(c, genasm::g_pair_cta, sizeof(unsigned) * n);
    static unsigned cs[8192];
    cudaMemcpyFromSymbol(cs, genasm::g_cta_sm, sizeof cs);
    for (int i = 0; i < n; ++i) out[2 * n + i] = c[i] | (unsigned long long)cs[c[i] % 8192] << 32;
}
extern "C" void ga_debug_timeline(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, genasm::g_timeline, sizeof(unsigned long long) * 512);
}
extern "C" void ga_debug_thread_stats(unsigned long long* out, int reset) {
    static unsigned long long w[genasm::kStatWarps][20];
    cudaMemcpyFromSymbol(w, genasm::g_wstats, sizeof w);
    cudaMemcpyFromSymbol(out, genasm::g_thread_stats, sizeof(unsigned long long) * 20);
    for (int k = 0; k < 20; ++k) {
        if (k == 6 || k == 7) continue;
        unsigned long long t = 0;
        for (int i = 0; i < genasm::kStatWarps; ++i) t += w[i][k];
        out[k] = t;
    }
    if (reset) {
        unsigned long long z[20] = {0, 0, 0, 0, 0, 0, ~0ull, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(genasm::g_thread_stats, z, sizeof z);
        static unsigned long long wz[genasm::kStatWarps][20];
        cudaMemcpyToSymbol(genasm::g_wstats, wz, sizeof wz);
        static unsigned long long tz[2][256];
        cudaMemcpyToSymbol(genasm::g_timeline, tz, sizeof tz);
        const unsigned long long big = ~0ull;
        cudaMemcpyToSymbol(genasm::g_t0, &big, sizeof big);
        static unsigned long long pz[262144];
        if (!pz[0]) for (auto& v : pz) v = ~0ull;
        cudaMemcpyToSymbol(genasm::g_pair_t, pz, sizeof pz);
    }
}
#endif
