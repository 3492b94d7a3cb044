// genasm_ws.cu -- warp-specialised fused GenASM-DC + GenASM-TB kernel (sm_100a).
//
// One CTA per SM.  Its warps split into
//   * DC warps: two groups of G = 16 lanes each.  Every group owns two window
//     SLOTS (double buffer) in shared memory and, each epoch, runs one DC pass
//     (levels-as-lanes wavefront, see DcLane) on one of them -- first building
//     the window's reversed chunks and pattern masks if the slot is fresh;
//   * TB warps: one LANE per slot.  Each lane owns its slot's pair state
//     (cursors, counters, output pointers), walks the traceback of a finished
//     window as a plain scalar loop over the band table (pkg/src/bitalign/
//     backtrace.py:113-160), advances the cursors (window.py:110-120), prepares
//     the next window or pulls the next pair from the global queue.
// A window that finishes its DC in epoch e is traced back in epoch e+1 while
// its group runs the other slot, so the wavefront never waits for the
// inherently serial traceback, and the traceback runs 16-32 windows at once
// with every lane busy instead of speculating along one diagonal.
//
// Slot ownership is a single state word: EMPTY/DONE belong to the TB lane,
// READY/IN_DC to the DC group.  Ownership moves by writing the state after a
// block-scope fence (release) and re-fencing after reading it (acquire); the
// epoch barrier (__syncthreads_or) doubles as the termination vote.
#include "genasm_device.cuh"

namespace genasm {

namespace {

enum : int { S_EMPTY = 0, S_READY = 1, S_DC = 2, S_DONE = 3 };

struct SlotMeta {
    const uint8_t* pchunk;  // P + p: the window's pattern chunk (forward)
    const uint8_t* tchunk;  // T + t: the window's text chunk (forward)
    int state, pass, full, d_min;
    int fail, m, n, budget;
};

constexpr int kG = 16;         // lanes per DC group
constexpr int kWsMaxBlock = 384;

template <int NW>
struct WsGeo {
    using GE = Geo<NW>;
    static constexpr int SLOT_W = GE::TAB_W + GE::WMAX * NW + GE::WMAX / 2;  // table, pm, codes
    static constexpr int CARRY_W = GE::WMAX * NW;
};

struct TbWalk {
    int d, j, i, consumed, tcons, wcost, no;
    unsigned lreads;
    bool stuck;
};

// The traceback walk of one window by one lane, up to column 0 (the caller
// applies the column-0 insertion rule).  Per state (d, j, i): edge bits from
// three table words (backtrace.py:84-99), first active edge by the priority
// LUT, then a branch-free state update.  FULLMODE reads full-width rows from
// the slot's global slab, otherwise the 32-bit band (or W <= 32 rows) in smem.
template <int NW, bool FULLMODE>
__device__ __forceinline__ void tb_walk(TbWalk& w, const uint32_t* __restrict__ tab,
                                        const uint32_t* __restrict__ gt,
                                        const uint8_t* __restrict__ cp,
                                        const uint8_t* __restrict__ ct, int m, int n, int W,
                                        int budget, uint64_t lut, uint8_t* __restrict__ out) {
    using GE = Geo<NW>;
    constexpr int WMAX = GE::WMAX;
    const int cbase = m - 1 - n - 15;  // band origin of column col: clamp(cbase + col)
    int d = w.d, j = w.j, i = w.i, consumed = w.consumed, tcons = w.tcons, wcost = w.wcost;
    int no = w.no;
    unsigned lreads = w.lreads;
    while (i >= 0 && consumed < budget && j > 0) {
        const int col1 = j - 1;
        const int dm1 = d > 0 ? d - 1 : 0;
        const int tcode = ct[col1];
        const int pcode = cp[i];
        uint32_t mb, sb, db, ib;  // table bits, 1 = inactive
        if (FULLMODE) {
            const int c = col1 > 1 ? col1 - 1 : 0;
            const int x0 = i > 0 ? i - 1 : 0;
            const uint32_t* rA = gt + ((int64_t)d * W + c) * NW;
            const uint32_t* rB = gt + ((int64_t)dm1 * W + c) * NW;
            const uint32_t* rU = gt + ((int64_t)dm1 * W + col1) * NW;
            mb = rA[x0 >> 5] >> (x0 & 31);
            sb = rB[x0 >> 5] >> (x0 & 31);
            db = rB[i >> 5] >> (i & 31);
            ib = rU[x0 >> 5] >> (x0 & 31);
        } else {
            const int c = col1 > 1 ? col1 - 1 : 0;
            const uint32_t A = tab[d * WMAX + c];
            const uint32_t Bd = tab[dm1 * WMAX + c];
            const uint32_t Bu = tab[dm1 * WMAX + col1];
            int a1 = cbase + col1;
            a1 = a1 < 0 ? 0 : (a1 > GE::BAND_MAX ? GE::BAND_MAX : a1);
            int a2 = cbase + j;
            a2 = a2 < 0 ? 0 : (a2 > GE::BAND_MAX ? GE::BAND_MAX : a2);
            mb = A >> (unsigned)(i - 1 - a1);
            sb = Bd >> (unsigned)(i - 1 - a1);
            db = Bd >> (unsigned)(i - a1);
            ib = Bu >> (unsigned)(i - 1 - a2);
        }
        if (col1 == 0) {  // column 0 is init(m, .): bit x inactive iff x >= level
            mb = i - 1 >= d;
            sb = i - 1 >= d - 1;
            db = i >= d - 1;
        }
        const unsigned dpos = d > 0;
        const unsigned i0 = i == 0;
        const unsigned mok = (unsigned)(tcode < 4) & (unsigned)(pcode == tcode) & (i0 | (~mb & 1u));
        const unsigned sok = dpos & (i0 | (~sb & 1u));
        const unsigned iok = dpos & (i0 | (~ib & 1u));
        const unsigned dok = dpos & (~db & 1u);
        const unsigned okm = mok | sok << 1 | iok << 2 | dok << 3;
        const unsigned op = (unsigned)(lut >> (4 * okm)) & 0xFu;
        if (op > OP_D) {
            w.stuck = true;
            break;
        }
        const unsigned j2 = j >= 2;
        lreads += j2 + (dpos ? j2 + 1u : 0u);
        // op in M,S,I,D = 0..3: j moves on M,S,D; d on S,I,D; i (and consumed) on M,S,I
        const int dj = (0xBu >> op) & 1u, dd = (0xEu >> op) & 1u, di = (0x7u >> op) & 1u;
        out[no++] = (uint8_t)(0x4449583Du >> (8 * op));  // "=XID"
        j -= dj;
        d -= dd;
        i -= di;
        consumed += di;
        tcons += dj;
        wcost += dd;
    }
    w.d = d;
    w.j = j;
    w.i = i;
    w.consumed = consumed;
    w.tcons = tcons;
    w.wcost = wcost;
    w.no = no;
    w.lreads = lreads;
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void vstore(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

template <int NW>
__global__ void __launch_bounds__(kWsMaxBlock, 1)
genasm_ws_kernel(const KernelParams P, const int nd) {
    constexpr int G = kG;
    using GE = Geo<NW>;
    using WG = WsGeo<NW>;
    constexpr int WMAX = GE::WMAX;
    constexpr bool BAND = GE::BAND;
    constexpr int LV = GE::LV;
    extern __shared__ __align__(16) uint32_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ngroups = nd * (32 / G);
    const int nslots = 2 * ngroups;
    const int ntb = (nslots + 31) / 32;
    uint32_t* slots = smem;
    uint32_t* carries = slots + nslots * WG::SLOT_W;
    SlotMeta* meta = reinterpret_cast<SlotMeta*>(carries + ngroups * WG::CARRY_W);
    const int W = P.W, O = P.O, K = P.k;
    auto slab = [&](int s) -> uint32_t* {
        return P.overflow + ((int64_t)blockIdx.x * nslots + s) * P.overflow_words_per_group;
    };

    if (warp < nd) {
        // ============================ DC warps ============================
        const int q = lane & (G - 1);
        const int gbase = lane & ~(G - 1);
        const unsigned lowmask = (1u << G) - 1u;
        const int group = warp * (32 / G) + lane / G;
        uint32_t* carry = carries + group * WG::CARRY_W;
        int cur = 0;
        for (;;) {
            if (!__syncthreads_or(0)) break;
            // ---- pick the slot: the current one if DC-owned, else the other ----
            int s = 2 * group + cur, st = S_EMPTY;
            if (q == 0) {
                st = vload(&meta[s].state);
                if (st != S_READY && st != S_DC) {
                    const int s2 = 2 * group + (cur ^ 1);
                    const int st2 = vload(&meta[s2].state);
                    if (st2 == S_READY || st2 == S_DC) {
                        s = s2;
                        st = st2;
                    }
                }
            }
            s = __shfl_sync(FULL, s, 0, G);
            st = __shfl_sync(FULL, st, 0, G);
            cur = s & 1;
            __threadfence_block();  // acquire: fields written before the state
            bool mine = st == S_READY || st == S_DC;
            SlotMeta& M = meta[s];
            uint32_t* tab = slots + s * WG::SLOT_W;
            uint32_t* pmcol = tab + GE::TAB_W;
            uint8_t* cp = reinterpret_cast<uint8_t*>(pmcol + WMAX * NW);
            uint8_t* ct = cp + WMAX;
            const int m = mine ? M.m : 1;
            const int n = mine ? M.n : 0;
            int pass = mine ? M.pass : 0;
            bool full = mine && M.full;

            // ---- fresh window: reversed chunks (window.py:99-100), masks (distance.py:70-94)
            if (__any_sync(FULL, mine && st == S_READY)) {
                const bool need = mine && st == S_READY;
                if (need) {
                    const uint8_t* pc = M.pchunk;
                    const uint8_t* tc = M.tchunk;
                    for (int i = q; i < m; i += G) cp[i] = pc[m - 1 - i];
                    for (int j = q; j < n; j += G) ct[j] = tc[n - 1 - j];
                }
                __syncwarp();
                uint32_t mt[4][NW];
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int w = 0; w < NW; ++w) mt[c][w] = 0u;
                if (need) {
                    for (int i = q; i < m; i += G) {
                        const int c = cp[i];
                        const uint32_t bit = 1u << (i & 31);
                        const int wi = i >> 5;
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                            for (int w = 0; w < NW; ++w) mt[cc][w] |= (c == cc && wi == w) ? bit : 0u;
                    }
                }
#pragma unroll
                for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                    for (int w = 0; w < NW; ++w) mt[cc][w] = ~group_or<G>(mt[cc][w]);
                if (need) {
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
                        __syncwarp(FULL >> (32 - G) << gbase);
                        if (q == 0) {
                            M.d_min = m;
                            M.fail = m > K;
                            __threadfence_block();
                            vstore(&M.state, S_DONE);
                        }
                        mine = false;
                        cur ^= 1;
                    }
                }
                __syncwarp();
            }

            // ---- one DC pass, both groups of the warp in lock-step ----
            const bool in_dc = mine;
            DcLane<NW, G> L;
            L.init(q, in_dc, pass, m, n, K, W, full, tab, carry, pmcol, slab(s));
            const int steps = __reduce_max_sync(FULL, in_dc ? n + G - 1 : 0);
            const int nmin = __reduce_min_sync(FULL, in_dc ? n : WMAX);
            const int fill_end = steps < G - 1 ? steps : G - 1;
            const int steady_end = nmin > fill_end ? nmin : fill_end;
            if (BAND && __any_sync(FULL, in_dc && full)) {
                for (int x = 0; x < fill_end; ++x) L.template step<true, true>(x);
                for (int x = fill_end; x < steady_end; ++x) L.template step<false, true>(x);
                for (int x = steady_end; x < steps; ++x) L.template step<true, true>(x);
            } else {
                for (int x = 0; x < fill_end; ++x) L.template step<true, false>(x);
#pragma unroll 4
                for (int x = fill_end; x < steady_end; ++x) L.template step<false, false>(x);
                for (int x = steady_end; x < steps; ++x) L.template step<true, false>(x);
            }
            const bool succ = L.active && n >= 1 &&
                              (word_sel<NW>(L.v, (m - 1) >> 5) & (1u << ((m - 1) & 31))) == 0u;
            const unsigned bal = (__ballot_sync(FULL, succ) >> gbase) & lowmask;
            __syncwarp();  // table and carry stores of the pass precede the hand-off
#ifdef GA_DEBUG
            if (in_dc && q == 0)
                printf("DC slot %d m=%d n=%d pass=%d full=%d bal=%x tchunk0=%d\n", s, m, n, pass,
                       (int)full, bal, (int)M.tchunk[0]);
#endif
            if (in_dc && q == 0) {
                int next = S_DC;
                if (bal) {
                    M.d_min = pass * G + __ffs(bal) - 1;
                    M.fail = 0;
                    next = S_DONE;
                } else if ((pass + 1) * G > K) {  // NotFound(k) -> WindowFailed(index, k)
                    M.fail = 1;
                    next = S_DONE;
                } else if (BAND && !full && (pass + 1) * G >= LV) {
                    M.full = 1;  // d_min > 15: the band cannot serve TB; redo full width
                    M.pass = 0;
                } else {
                    M.pass = pass + 1;
                }
                M.full = next == S_DC ? M.full : (int)full;
                __threadfence_block();
                vstore(&M.state, next == S_DONE ? S_DONE : S_DC);
            }
            if (in_dc && (bal || (pass + 1) * G > K)) cur ^= 1;
        }
        return;
    }

    // ============================ TB warps ============================
    // slot s is served by TB warp s % ntb, lane s / ntb
    const int tw = warp - nd;
    const int s = lane * ntb + tw;
    const bool own = s < nslots;
    SlotMeta& M = meta[own ? s : 0];
    uint32_t* tab = slots + (own ? s : 0) * WG::SLOT_W;
    const uint8_t* cp = reinterpret_cast<const uint8_t*>(tab + GE::TAB_W + WMAX * NW);
    const uint8_t* ct = cp + WMAX;
    uint32_t* gt = slab(own ? s : 0);
    PairResult* results = reinterpret_cast<PairResult*>(P.results);
    // pair state of this slot
    int64_t pair = -1, p = 0, t = 0, nops = 0;
    int Lp = 0, Lt = 0, widx = 0, m = 0, n = 0, budget = 0;
    const uint8_t* Pp = nullptr;
    const uint8_t* Tp = nullptr;
    uint8_t* ops = nullptr;
    uint8_t* dists = nullptr;
    int64_t cost = 0, rows = 0, reads = 0, writes = 0, words = 0;
    bool exhausted = false;
    if (own) {
        M.state = S_EMPTY;
        M.pass = M.full = M.fail = 0;
    }

    auto finish = [&](int status, int fail_window) {
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
    };
    // next window's geometry (window.py:96-101) -> slot meta; returns READY
    auto prepare = [&]() -> int {
        const int64_t remaining = Lp - p;
        const bool final_w = remaining <= W;
        m = final_w ? (int)remaining : W;
        const int64_t tleft = Lt - t;
        n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
        budget = final_w ? m : W - O;
        M.pchunk = Pp + p;
        M.tchunk = Tp + t;
        M.m = m;
        M.n = n;
        M.budget = budget;
        M.pass = 0;
        M.full = 0;
        M.fail = 0;
        return S_READY;
    };

    for (;;) {
        if (own) {
            const int st0 = vload(&M.state);
            int st = st0;
            if (st == S_DONE) {
                __threadfence_block();  // acquire the DC group's table and fields
                const int d_min = M.d_min;
                if (M.fail) {
                    finish(1, widx);
                    st = S_EMPTY;
                } else {
                    // ---- scalar traceback (backtrace.py:113-160) ----
                    TbWalk w;
                    w.d = d_min;
                    w.j = n;
                    w.i = m - 1;
                    w.consumed = w.tcons = w.wcost = w.no = 0;
                    w.lreads = 0;
                    w.stuck = false;
                    uint8_t* out = ops + nops;
                    if (BAND && M.full) {
                        tb_walk<NW, true>(w, tab, gt, cp, ct, m, n, W, budget, P.prio_lut, out);
                    } else {
                        tb_walk<NW, false>(w, tab, gt, cp, ct, m, n, W, budget, P.prio_lut, out);
                    }
                    // column 0 (reached with pattern and budget left): the init zeros
                    // cover i+1 insertions at level d (backtrace.py:122-132)
                    if (!w.stuck && w.i >= 0 && w.consumed < budget && w.j == 0) {
                        if (w.i + 1 > w.d) {
                            w.stuck = true;
                        } else {
                            const int left = budget - w.consumed;
                            const int take = w.i + 1 < left ? w.i + 1 : left;
                            for (int u = 0; u < take; ++u) out[w.no + u] = 'I';
                            w.no += take;
                            w.wcost += take;
                            w.consumed += take;
                            w.i -= take;
                        }
                    }
                    const bool stuck = w.stuck;
                    const int consumed = w.consumed, tcons = w.tcons, wcost = w.wcost, no = w.no;
                    const unsigned lreads = w.lreads;
#ifdef GA_DEBUG
                    printf("TB slot %d widx=%d d_min=%d full=%d m=%d n=%d consumed=%d tcons=%d stuck=%d\n",
                           s, widx, d_min, M.full, m, n, consumed, tcons, (int)stuck);
#endif
                    if (stuck) {
                        finish(3, widx);
                        st = S_EMPTY;
                    } else {
                        // closed-form entry_writes (dptable.py:62-82, 156-171)
                        int64_t wr = 0;
                        for (int dd = 0; dd <= d_min; ++dd) {
                            int ss = n - budget - (K - dd) - 1;
                            ss = ss > 1 ? ss : 1;
                            const int cnt = n - ss + 1;
                            wr += cnt > 0 ? cnt : 0;
                        }
                        dists[widx] = (uint8_t)d_min;
                        rows += d_min + 1;
                        cost += wcost;
                        reads += lreads;
                        writes += wr;
                        words += wr * ((m + 63) / 64);
                        nops += no;
                        p += consumed;
                        t += tcons;
                        ++widx;
                        if (p < Lp) {
                            st = prepare();
                        } else {
                            finish(0, -1);
                            st = S_EMPTY;
                        }
                    }
                }
            }
            // ---- refill an empty slot from the global queue (empty patterns settle here)
            while (st == S_EMPTY && !exhausted) {
                const unsigned long long idx = atomicAdd(P.queue, 1ull);
                if (idx >= (unsigned long long)P.n_pairs) {
                    exhausted = true;
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
                if (Lp <= 0) {
                    finish(2, -1);  // EmptyPattern (window.py:87-88)
                } else {
                    st = prepare();
                }
            }
            // hand a TB-owned slot back (never touch a slot the DC group owns)
            if (st0 == S_DONE || st0 == S_EMPTY) {
                __threadfence_block();  // release the fields before the state
                vstore(&M.state, st);
            }
        }
        const int alive = own && vload(&M.state) != S_EMPTY;
        if (!__syncthreads_or(alive)) break;
    }
}

}  // namespace

template <int NW>
static cudaError_t launch_ws_t(const KernelParams& base, int nd_req, int num_sms,
                               cudaStream_t stream, uint32_t** overflow, size_t* overflow_cap,
                               LaunchShape* shape) {
    using GE = Geo<NW>;
    using WG = WsGeo<NW>;
    KernelParams P = base;
    // shared memory per DC warp: 4 slots + 2 carry rows + 4 slot records
    const int per_dc_warp = 4 * WG::SLOT_W * 4 + 2 * WG::CARRY_W * 4 + 4 * (int)sizeof(SlotMeta);
    const int budget = 225 * 1024;
    int nd = budget / per_dc_warp;
    if (nd_req > 0 && nd_req < nd) nd = nd_req;
    if (nd > 10) nd = 10;
    if (nd < 1) return cudaErrorInvalidConfiguration;
    const int nslots = 4 * nd;
    const int ntb = (nslots + 31) / 32;
    const int block = (nd + ntb) * 32;
    const int smem = nd * per_dc_warp;
    auto kern = genasm_ws_kernel<NW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int grid = num_sms * per_sm;
    const int64_t max_useful = (P.n_pairs + nslots - 1) / nslots;
    if (grid > max_useful) grid = (int)(max_useful > 0 ? max_useful : 1);
    const int levels_cap = ((P.k + 1 + kG - 1) / kG) * kG;
    P.overflow_words_per_group = GE::BAND ? (int64_t)levels_cap * P.W * NW : 0;
    const size_t need = (size_t)grid * nslots * (size_t)P.overflow_words_per_group;
    if (need > *overflow_cap || !*overflow) {
        if (*overflow) cudaFree(*overflow);
        *overflow = nullptr;
        *overflow_cap = 0;
        e = cudaMalloc(overflow, need * 4 + 64);
        if (e != cudaSuccess) return e;
        *overflow_cap = need;
    }
    P.overflow = *overflow;
    kern<<<grid, block, smem, stream>>>(P, nd);
    shape->grid = grid;
    shape->block = block;
    shape->smem_bytes = smem;
    shape->group = kG;
    shape->blocks_per_sm = per_sm;
    shape->overflow_words_per_group = P.overflow_words_per_group;
    return cudaGetLastError();
}

cudaError_t launch_genasm_ws(const KernelParams& P, int dc_warps, int num_sms, cudaStream_t stream,
                             uint32_t** overflow, size_t* cap, LaunchShape* shape) {
    if (P.W <= 32) return launch_ws_t<1>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_ws_t<2>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_ws_t<4>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm
