// genasm_pipeline.cu -- warp-specialised fused GenASM-DC + GenASM-TB kernel (sm_100a).
//
// One CTA per SM; its warps split into
//   * DC warps: two groups of G = 16 lanes each.  Every group owns two window
//     SLOTS (double buffer) in shared memory and, each epoch, runs one DC pass
//     (levels-as-lanes wavefront, see DcLane) on one of them -- first building
//     the window's reversed chunks and pattern masks if the slot is fresh;
//   * TB warps: four traceback groups of 8 lanes each.  Every slot belongs to
//     one TB group, which walks the traceback of its finished windows with the
//     8 lanes speculating 8 diagonal ('=') states per round
//     (pkg/src/bitalign/backtrace.py:113-160), advances the pair cursors
//     (window.py:110-120), prepares the next window or pulls the next pair.
// A window whose DC ends in epoch e is traced back in epoch e+1 while its DC
// group runs the other slot, so the wavefront never waits for the serial
// traceback and the traceback never stalls the wavefront's warps.
//
// Slot ownership is a single state word: EMPTY/DONE belong to the TB group,
// READY/IN_DC to the DC group.  Ownership moves by writing the state after a
// block-scope fence (release) and fencing after reading it (acquire); the
// epoch barrier (__syncthreads_or) doubles as the termination vote.
#include "genasm_device.cuh"

namespace genasm {

namespace {

enum : int { S_EMPTY = 0, S_READY = 1, S_DC = 2, S_DONE = 3 };

struct SlotMeta {
    // the window (written by the TB group, read by the DC group)
    const uint8_t* pchunk;  // P + p: the window's pattern chunk (forward)
    const uint8_t* tchunk;  // T + t: the window's text chunk (forward)
    int state, pass, full, d_min;
    int fail, m, n, budget;
    // the pair (TB group only)
    const uint8_t* Pp;
    const uint8_t* Tp;
    uint8_t* ops;
    uint8_t* dists;
    long long pair, p, t, nops, cost, rows, reads, writes, words;
    int Lp, Lt, widx, pad;
};

constexpr int kG = 16;   // lanes per DC group
#ifndef GA_TB_LANES
#define GA_TB_LANES 4
#endif
constexpr int kTG = GA_TB_LANES;  // lanes per TB group (one slot each)
constexpr int kPipeMaxBlock = 768;

template <int NW>
struct WsGeo {
    using GE = Geo<NW>;
    static constexpr int SLOT_W = GE::TAB_W + GE::WMAX * NW + GE::WMAX / 2;  // table, pm, codes
    static constexpr int CARRY_W = GE::WMAX * NW;
};

#ifdef GA_PROFILE
// [0] DC epoch cycles (per DC warp) [1] DC epochs [2] TB work cycles (per TB warp)
// [3] TB epochs [4] TB cycles waiting at the epoch barrier [5] pass cycles [6] pass steps
__device__ unsigned long long g_prof[8];
#endif

struct TbWalk {
    int d, j, i, consumed, tcons, wcost, no;
    unsigned lreads;  // per lane
    bool stuck;
};

// Speculative traceback of one window per TG-lane group (backtrace.py:113-160).
// All 32 lanes call it; `going` is group-uniform.  Lane q evaluates the state
// q diagonal ('=') steps ahead: edge bits from three table words
// (backtrace.py:84-99) and the chunk codes, the chosen edge by the priority
// LUT.  A ballot finds the first lane whose edge is not '=' (or that stops);
// the group takes the '=' run plus that lane's edge in one round.  Ops go to
// `out` in walk (= forward) order; the column-0 insertion rule ends the walk.
template <int NW, int TG>
__device__ __forceinline__ void tb_spec(TbWalk& w, bool going, int q, int gbase, bool full,
                                        const uint32_t* __restrict__ tab,
                                        const uint32_t* __restrict__ gt,
                                        const uint8_t* __restrict__ cp,
                                        const uint8_t* __restrict__ ct, int m, int n, int W,
                                        int budget, uint32_t lut_lo, uint32_t lut_hi,
                                        uint8_t* __restrict__ out) {
    using GE = Geo<NW>;
    constexpr int WMAX = GE::WMAX;
    constexpr unsigned lowmask = (1u << TG) - 1u;
    const int cbase = m - 1 - n - 15;  // band origin of column col: clamp(cbase + col)
    int d = w.d, j = w.j, i = w.i, consumed = 0, tcons = 0, wcost = 0, no = 0;
    unsigned lreads = 0;
    bool stuck = false;
    for (;;) {
        if (going) {
            if (i < 0 || consumed >= budget) {
                going = false;
            } else if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
                if (i + 1 > d) {
                    stuck = true;
                } else {
                    const int left = budget - consumed;
                    const int take = i + 1 < left ? i + 1 : left;
                    for (int u = q; u < take; u += TG) out[no + u] = 'I';
                    no += take;
                    wcost += take;
                    consumed += take;
                    i -= take;
                }
                going = false;
            }
        }
        if (!__any_sync(FULL, going)) break;
        const int jq = j - q, iq = i - q;
        int op = OP_STOP;
        unsigned rd = 0;
        if (going && iq >= 0 && consumed + q < budget && jq >= 1) {
            const int col1 = jq - 1;
            const int dm1 = d > 0 ? d - 1 : 0;
            const int c = col1 > 1 ? col1 - 1 : 0;
            const int tcode = ct[col1];
            const int pcode = cp[iq];
            uint32_t mb, sb, db, ib;  // table bits, 1 = inactive
            if (full) {
                const int x0 = iq > 0 ? iq - 1 : 0;
                const uint32_t* rA = gt + ((int64_t)d * W + c) * NW;
                const uint32_t* rB = gt + ((int64_t)dm1 * W + c) * NW;
                const uint32_t* rU = gt + ((int64_t)dm1 * W + col1) * NW;
                mb = rA[x0 >> 5] >> (x0 & 31);
                sb = rB[x0 >> 5] >> (x0 & 31);
                db = rB[iq >> 5] >> (iq & 31);
                ib = rU[x0 >> 5] >> (x0 & 31);
            } else {
                const uint32_t A = tab[d * WMAX + c];
                const uint32_t Bd = tab[dm1 * WMAX + c];
                const uint32_t Bu = tab[dm1 * WMAX + col1];
                int a1 = cbase + col1;
                a1 = a1 < 0 ? 0 : (a1 > GE::BAND_MAX ? GE::BAND_MAX : a1);
                int a2 = cbase + jq;
                a2 = a2 < 0 ? 0 : (a2 > GE::BAND_MAX ? GE::BAND_MAX : a2);
                mb = A >> (unsigned)(iq - 1 - a1);
                sb = Bd >> (unsigned)(iq - 1 - a1);
                db = Bd >> (unsigned)(iq - a1);
                ib = Bu >> (unsigned)(iq - 1 - a2);
            }
            if (col1 == 0) {  // column 0 is init(m, .): bit x inactive iff x >= level
                mb = iq - 1 >= d;
                sb = iq - 1 >= d - 1;
                db = iq >= d - 1;
            }
            const unsigned dpos = d > 0;
            const unsigned i0 = iq == 0;
            const unsigned mok = (unsigned)(tcode < 4) & (unsigned)(pcode == tcode) &
                                 (i0 | (~mb & 1u));
            const unsigned sok = dpos & (i0 | (~sb & 1u));
            const unsigned iok = dpos & (i0 | (~ib & 1u));
            const unsigned dok = dpos & (~db & 1u);
            const unsigned okm = mok | sok << 1 | iok << 2 | dok << 3;
            op = (int)(((okm & 8u) ? lut_hi : lut_lo) >> (4u * (okm & 7u))) & 0xF;
            const unsigned j2 = jq >= 2;
            rd = j2 + (dpos ? j2 + 1u : 0u);
        }
        const unsigned nz = (__ballot_sync(FULL, op != OP_M) >> gbase) & lowmask;
        const int f = nz ? __ffs(nz) - 1 : TG;
        const int opf = __shfl_sync(FULL, op, f & (TG - 1), TG);
        if (going) {
            if (q < f) {
                out[no + q] = '=';
                lreads += rd;
            }
            j -= f;
            i -= f;
            consumed += f;
            tcons += f;
            no += f;
            if (f < TG && opf != OP_STOP) {
                if (opf == OP_STUCK) {
                    stuck = true;
                    going = false;
                } else {
                    if (q == f) lreads += rd;
                    // op in S,I,D = 1..3: j moves on S,D; i (consumed) on S,I; d on all
                    const int dj = (0xBu >> opf) & 1u, di = (0x7u >> opf) & 1u;
                    if (q == 0) out[no] = (uint8_t)(0x4449583Du >> (8 * opf));  // "=XID"
                    ++no;
                    ++wcost;
                    j -= dj;
                    --d;
                    i -= di;
                    consumed += di;
                    tcons += dj;
                }
            }
        }
    }
    w.d = d;
    w.j = j;
    w.i = i;
    w.consumed = consumed;
    w.tcons = tcons;
    w.wcost = wcost;
    w.no = no;
    w.lreads = lreads;
    w.stuck = stuck;
}

__device__ __forceinline__ int vload(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void vstore(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }

template <int NW>
__global__ void __launch_bounds__(kPipeMaxBlock, 1)
genasm_pipeline_kernel(const KernelParams P, const int nd, const int nt) {
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
#ifdef GA_PROFILE
            const long long t_epoch0 = clock64();
#endif
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
#ifdef GA_PROFILE
            const long long t_pass0 = clock64();
#endif
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
#ifdef GA_PROFILE
            if (lane == 0 && steps > 0) {
                atomicAdd(&g_prof[5], (unsigned long long)(clock64() - t_pass0));
                atomicAdd(&g_prof[6], (unsigned long long)steps);
            }
#endif
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
#ifdef GA_PROFILE
            if (lane == 0) {
                atomicAdd(&g_prof[0], (unsigned long long)(clock64() - t_epoch0));
                atomicAdd(&g_prof[1], 1ull);
            }
#endif
        }
        return;
    }

    // ============================ TB warps ============================
    // TB group tg (8 lanes) serves slots tg, tg + ntg, ...
    const int tq = lane & (kTG - 1);
    const int tgbase = lane & ~(kTG - 1);
    const int tg = (warp - nd) * (32 / kTG) + lane / kTG;
    const int ntg = nt * (32 / kTG);
    const int kmax = (nslots + ntg - 1) / ntg;
    const uint32_t lut_lo = (uint32_t)P.prio_lut, lut_hi = (uint32_t)(P.prio_lut >> 32);
    PairResult* results = reinterpret_cast<PairResult*>(P.results);
    bool exhausted = false;  // lane tq == 0 of each TB group
    for (int k = 0; k < kmax; ++k) {
        const int s = tg + k * ntg;
        if (s < nslots && tq == 0) {
            meta[s].state = S_EMPTY;
            meta[s].pass = meta[s].full = meta[s].fail = 0;
        }
    }
    __syncwarp();

    for (;;) {
#ifdef GA_PROFILE
        const long long t_tb0 = clock64();
#endif
        int alive = 0;
        for (int k = 0; k < kmax; ++k) {
            const int s = tg + k * ntg;
            const bool own = s < nslots;
            SlotMeta& M = meta[own ? s : 0];
            int st0 = own && tq == 0 ? vload(&M.state) : S_READY;
            st0 = __shfl_sync(FULL, st0, 0, kTG);
            __threadfence_block();  // acquire the DC group's table and fields
            const bool done = st0 == S_DONE;
            const bool walk = done && !M.fail;
            uint32_t* tab = slots + (own ? s : 0) * WG::SLOT_W;
            const uint8_t* cp = reinterpret_cast<const uint8_t*>(tab + GE::TAB_W + WMAX * NW);
            const uint8_t* ct = cp + WMAX;
            const int m = M.m, n = M.n, budget = M.budget, d_min = M.d_min;
            TbWalk w;
            w.d = d_min;
            w.j = n;
            w.i = m - 1;
            tb_spec<NW, kTG>(w, walk, tq, tgbase, BAND && M.full, tab, slab(own ? s : 0), cp, ct,
                             m, n, W, budget, lut_lo, lut_hi, M.ops + M.nops);
            // closed-form entry_writes (dptable.py:62-82, 156-171)
            unsigned wr = 0;
            if (walk && !w.stuck) {
                for (int dd = tq; dd <= d_min; dd += kTG) {
                    int ss = n - budget - (K - dd) - 1;
                    ss = ss > 1 ? ss : 1;
                    const int cnt = n - ss + 1;
                    wr += cnt > 0 ? (unsigned)cnt : 0u;
                }
            }
            wr = group_sum<kTG>(wr);
            const unsigned lreads = group_sum<kTG>(w.lreads);
            if (own && tq == 0 && (done || st0 == S_EMPTY)) {
                int st = st0;
                auto finish = [&](int status) {
                    PairResult r{};
                    r.status = status;
                    r.fail_window = status == 0 || status == 2 ? -1 : M.widx;
                    if (status == 0) {
                        r.cost = M.cost;
                        r.text_consumed = M.t;
                        r.rows_computed = M.rows;
                        r.ops_len = M.nops;
                        r.entry_reads = M.reads;
                        r.entry_writes = M.writes;
                        r.words_allocated = M.words;
                    }
                    results[M.pair] = r;
                };
                // next window's geometry (window.py:96-101)
                auto prepare = [&]() -> int {
                    const long long remaining = M.Lp - M.p;
                    const bool final_w = remaining <= W;
                    const int mm = final_w ? (int)remaining : W;
                    const long long tleft = M.Lt - M.t;
                    M.pchunk = M.Pp + M.p;
                    M.tchunk = M.Tp + M.t;
                    M.m = mm;
                    M.n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
                    M.budget = final_w ? mm : W - O;
                    M.pass = 0;
                    M.full = 0;
                    M.fail = 0;
                    return S_READY;
                };
                if (done) {
                    if (M.fail) {
                        finish(1);  // NotFound(k) -> WindowFailed(index, k)
                        st = S_EMPTY;
                    } else if (w.stuck) {
                        finish(3);
                        st = S_EMPTY;
                    } else {
                        M.dists[M.widx] = (uint8_t)d_min;
                        M.rows += d_min + 1;
                        M.cost += w.wcost;
                        M.reads += lreads;
                        M.writes += wr;
                        M.words += (long long)wr * ((m + 63) / 64);
                        M.nops += w.no;
                        M.p += w.consumed;
                        M.t += w.tcons;
                        M.widx += 1;
                        if (M.p < M.Lp) {
                            st = prepare();
                        } else {
                            finish(0);
                            st = S_EMPTY;
                        }
                    }
                }
                // refill from the global queue (empty patterns settle here)
                while (st == S_EMPTY && !exhausted) {
                    const unsigned long long idx = atomicAdd(P.queue, 1ull);
                    if (idx >= (unsigned long long)P.n_pairs) {
                        exhausted = true;
                        break;
                    }
                    const long long pair = P.order ? (long long)P.order[idx] : (long long)idx;
                    M.pair = pair;
                    M.Lp = P.pat_len[pair];
                    M.Lt = P.txt_len[pair];
                    M.Pp = P.codes + P.pat_off[pair];
                    M.Tp = P.codes + P.txt_off[pair];
                    M.ops = P.ops + P.ops_off[pair];
                    M.dists = P.dists + P.win_off[pair];
                    M.p = M.t = M.nops = 0;
                    M.widx = 0;
                    M.cost = M.rows = M.reads = M.writes = M.words = 0;
                    if (M.Lp <= 0) {
                        finish(2);  // EmptyPattern (window.py:87-88)
                    } else {
                        st = prepare();
                    }
                }
                __threadfence_block();  // release the fields before the state
                vstore(&M.state, st);
            }
            if (own && tq == 0) alive |= vload(&M.state) != S_EMPTY;
            __syncwarp();
        }
#ifdef GA_PROFILE
        if (lane == 0) {
            atomicAdd(&g_prof[2], (unsigned long long)(clock64() - t_tb0));
            atomicAdd(&g_prof[3], 1ull);
        }
        const long long t_bar0 = clock64();
#endif
        if (!__syncthreads_or(alive)) break;
#ifdef GA_PROFILE
        if (lane == 0) atomicAdd(&g_prof[4], (unsigned long long)(clock64() - t_bar0));
#endif
    }
}

}  // namespace

template <int NW>
static cudaError_t launch_pipe_t(const KernelParams& base, int nd_req, int num_sms,
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
    if (nd > 12) nd = 12;
    if (nd < 1) return cudaErrorInvalidConfiguration;
    // one TB group per slot: nt warps of 32/kTG groups serve the 4*nd slots
    auto tb_warps = [](int ndw) { return (4 * ndw + 32 / kTG - 1) / (32 / kTG); };
    while (nd > 1 && (nd + tb_warps(nd)) * 32 > kPipeMaxBlock) --nd;
    const int nslots = 4 * nd;
    const int nt = tb_warps(nd);
    const int block = (nd + nt) * 32;
    const int smem = nd * per_dc_warp;
    auto kern = genasm_pipeline_kernel<NW>;
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
    kern<<<grid, block, smem, stream>>>(P, nd, nt);
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
    if (P.W <= 32) return launch_pipe_t<1>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_pipe_t<2>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_pipe_t<4>(P, dc_warps, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm

#ifdef GA_PROFILE
extern "C" void ga_debug_prof(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, genasm::g_prof, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(genasm::g_prof, z, sizeof z);
    }
}
#endif
