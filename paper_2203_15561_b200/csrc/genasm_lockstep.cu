// genasm_lockstep.cu -- the fused windowed DC+TB kernel (sm_100a): every group
// of G lanes owns one pair and runs DC, traceback and window setup itself;
// the groups of a warp advance in pass rounds.  Design: genasm_kernel.cuh.
#include "genasm_device.cuh"

namespace genasm {

template <int NW, int G>
__host__ __device__ constexpr int smem_pad() {
    return G * NW > 32 ? G * NW : 32;
}

template <int NW, int G, int LPL>
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
    const unsigned lowmask = (G == 32) ? FULL : ((1u << G) - 1u);
    const int gib = threadIdx.x / G;
    const int groups_per_block = blockDim.x / G;

    constexpr int LPP = G * LPL;                       // levels per pass
    constexpr int SMAX = WMAX + G - 1;                 // wavefront steps per pass
    constexpr int NPASS = BAND ? 1 : (LV + LPP - 1) / LPP;  // band-table passes
    // pads: the wavefront's look-ahead loads reach G*NW words before a group's
    // region and past its end (smem_pad<>)
    uint32_t* carry = smem + smem_pad<NW, G>() + gib * (2 * WMAX * NW + WMAX / 2);
    uint32_t* pmcol = carry + WMAX * NW;
    uint8_t* cp = reinterpret_cast<uint8_t*>(pmcol + WMAX * NW);
    uint8_t* ct = cp + WMAX;
    const int64_t gid = (int64_t)blockIdx.x * groups_per_block + gib;
    uint32_t* gtab = P.overflow + gid * P.overflow_words_per_group;
    // this warp's band table: [pass][step][lane][LPL] words (DcLaneM)
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t* gband = P.band + wid * (int64_t)NPASS * SMAX * 32 * LPL;
    // band word of table entry (level e, column index c = col-1): written by lane
    // q = (e mod LPP) / LPL of the group at step c + q of pass e / LPP
    auto bword = [&](int e, int c) -> uint32_t {
        const int pp = e / LPP, r = e - pp * LPP, qq = r / LPL, kk = r - qq * LPL;
        return gband[(((int64_t)pp * SMAX + c + qq) * 32 + gbase + qq) * LPL + kk];
    };
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

    // called by all G lanes of the group
    const unsigned long long n_eff = (unsigned long long)P.n_pairs;

    auto write_result = [&](int status, int fail_window) {
        if (status == 1 || status == 3) {  // windows the pair never completed read as 0
            const int64_t step = W - O;
            const int64_t nwin = Lp <= W ? 1 : 1 + (Lp - W + step - 1) / step;
            for (int64_t i = fail_window + q; i < nwin; i += G) dists[i] = 0;
        }
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

    for (;;) {
        // ================= next pair (empty patterns are settled here) =================
        while (__any_sync(FULL, phase == NEED_PAIR)) {
            const bool need = phase == NEED_PAIR;
            unsigned long long idx = 0;
            if (need && q == 0) idx = atomicAdd(P.queue, 1ull);
            idx = __shfl_sync(FULL, idx, 0, G);
            if (need) {
                if (idx >= n_eff) {
                    phase = DONE;
                } else {
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
                    if (Lp <= 0) write_result(2, -1);  // EmptyPattern (window.py:87-88)
                    else phase = NEED_WINDOW;
                }
            }
        }
        if (__all_sync(FULL, phase == DONE)) break;

        // ================= next window: geometry, chunks, masks =================
        if (__any_sync(FULL, phase == NEED_WINDOW)) {
            const bool need = phase == NEED_WINDOW;
            if (need) {
                // window geometry (window.py:96-101)
                const int64_t remaining = Lp - p;
                const bool final_w = remaining <= W;
                m = final_w ? (int)remaining : W;
                const int64_t tleft = Lt - t;
                n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
                budget = final_w ? m : W - O;
                // reversed chunks (window.py:99-100)
                for (int i = q; i < m; i += G) cp[i] = Pp[p + m - 1 - i];
                for (int j = q; j < n; j += G) ct[j] = Tp[t + n - 1 - j];
            }
            __syncwarp();
            // pattern masks (distance.py:70-79): match bits per symbol, OR-reduced
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
                // per-column masks (distance.py:91-94): PM[T[j-1]], all-ones off the alphabet
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
            __syncwarp();
        }

        // ================= DC pass round (all groups in lock-step) =================
        {
            const bool in_dc = phase == IN_DC;
            DcLaneM<NW, G, LPL> L;
            L.init(q, in_dc, pass, m, n, K, W, full, const_cast<uint32_t*>(gband), lane, carry,
                   pmcol, gtab);
            // warp-uniform trip counts: fill [0, G-1), steady [G-1, nmin), drain [.., steps)
            const int steps = __reduce_max_sync(FULL, in_dc ? n + G - 1 : 0);
            const int nmin = __reduce_min_sync(FULL, in_dc ? n : WMAX);
            const int fill_end = steps < G - 1 ? steps : G - 1;
            const int steady_end = nmin > fill_end ? nmin : fill_end;
            if (BAND && __any_sync(FULL, in_dc && full)) {
                for (int s = 0; s < fill_end; ++s) L.template step<true, true>(s);
                for (int s = fill_end; s < steady_end; ++s) L.template step<false, true>(s);
                for (int s = steady_end; s < steps; ++s) L.template step<true, true>(s);
            } else {
                for (int s = 0; s < fill_end; ++s) L.template step<true, false>(s);
#pragma unroll 4
                for (int s = fill_end; s < steady_end; ++s) L.template step<false, false>(s);
                for (int s = steady_end; s < steps; ++s) L.template step<true, false>(s);
            }
            const int fs = L.first_success(m);
            const unsigned bal = (__ballot_sync(FULL, fs >= 0) >> gbase) & lowmask;
            const int lq = bal ? __ffs(bal) - 1 : 0;  // lowest lane holding a solved level
            const int fsl = __shfl_sync(FULL, fs, lq, G);
            if (in_dc) {
                if (bal) {
                    d_min = pass * LPP + lq * LPL + fsl;
                    phase = IN_TB;
                } else if ((pass + 1) * LPP > K) {  // NotFound(k) -> WindowFailed(index, k)
                    write_result(1, widx);
                    phase = NEED_PAIR;
                } else if (BAND && !full && (pass + 1) * LPP >= LV) {
                    full = true;  // d_min > 15: the band cannot serve TB; redo full width
                    pass = 0;
                } else {
                    ++pass;
                }
            }
        }

        // ================= TB round (groups whose window solved) =================
        if (__any_sync(FULL, phase == IN_TB)) {
            __syncwarp();
            const bool tbg = phase == IN_TB;
            int d = d_min, j = n, i = m - 1, consumed = 0, tcons = 0, wcost = 0;
            unsigned lreads = 0;
            bool stuck = false, going = tbg;
            const int cbase = m - 1 - n - 15;  // band origin of column col: cbase + col, clamped
            for (;;) {
                if (going) {
                    if (i < 0 || consumed >= budget) {
                        going = false;
                    } else if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
                        if (i + 1 > d) {
                            stuck = true;
                        } else {
                            const int take = (i + 1 < budget - consumed) ? i + 1 : budget - consumed;
                            for (int u = q; u < take; u += G) ops[nops + u] = 'I';
                            nops += take;
                            wcost += take;
                            consumed += take;
                            i -= take;
                        }
                        going = false;
                    }
                }
                if (!__any_sync(FULL, going)) break;
                // lane q evaluates the state q diagonal ('=') steps ahead (backtrace.py:88-99)
                const int jq = j - q, iq = i - q;
                int op = OP_STOP;
                unsigned rd = 0;
                if (going && iq >= 0 && consumed + q < budget && jq >= 1) {
                    const int tcode = ct[jq - 1];
                    const bool symeq = tcode < 4 && cp[iq] == tcode;
                    const int dm1 = d > 0 ? d - 1 : 0;
                    const int col1 = jq - 1;
                    uint32_t mb, sb, db, ib;  // table bits, 1 = inactive
                    if (BAND && full) {
                        auto gbit = [&](int e, int col, int x) -> uint32_t {
                            col = col > 1 ? col : 1;
                            x = x > 0 ? x : 0;
                            const uint32_t* row = gtab + ((int64_t)e * W + (col - 1)) * NW;
                            return row[x >> 5] >> (x & 31);
                        };
                        mb = gbit(d, col1, iq - 1);
                        sb = gbit(dm1, col1, iq - 1);
                        db = gbit(dm1, col1, iq);
                        ib = gbit(dm1, jq, iq - 1);
                    } else {
                        const int c1 = col1 > 1 ? col1 - 1 : 0;
                        const uint32_t A = bword(d, c1);
                        const uint32_t Bd = bword(dm1, c1);
                        const uint32_t Bu = bword(dm1, jq - 1);
                        int a1 = cbase + col1, a2 = cbase + jq;
                        a1 = a1 < 0 ? 0 : (a1 > GE::BAND_MAX ? GE::BAND_MAX : a1);
                        a2 = a2 < 0 ? 0 : (a2 > GE::BAND_MAX ? GE::BAND_MAX : a2);
                        mb = A >> (unsigned)(iq - 1 - a1);
                        sb = Bd >> (unsigned)(iq - 1 - a1);
                        db = Bd >> (unsigned)(iq - a1);
                        ib = Bu >> (unsigned)(iq - 1 - a2);
                    }
                    if (jq == 1) {  // column 0 is init(m, .): bit x inactive iff x >= level
                        mb = iq - 1 >= d;
                        sb = iq - 1 >= d - 1;
                        db = iq >= d - 1;
                    }
                    const bool mok = symeq && (iq == 0 || !(mb & 1u));
                    const bool dpos = d > 0;
                    const bool sok = dpos && (iq == 0 || !(sb & 1u));
                    const bool iok = dpos && (iq == 0 || !(ib & 1u));
                    const bool dok = dpos && !(db & 1u);
                    const unsigned okm = (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 |
                                         (unsigned)dok << 3;
                    op = (int)((P.prio_lut >> (4 * okm)) & 0xFu);
                    rd = (unsigned)(jq >= 2) + (dpos ? (unsigned)(jq >= 2) + 1u : 0u);
                }
                const unsigned nz = (__ballot_sync(FULL, op != OP_M) >> gbase) & lowmask;
                const int f = nz ? __ffs(nz) - 1 : G;
                const int opf = __shfl_sync(FULL, op, f & (G - 1), G);
                if (going) {
                    if (q < f) {
                        ops[nops + q] = '=';
                        lreads += rd;
                    }
                    j -= f;
                    i -= f;
                    consumed += f;
                    tcons += f;
                    nops += f;
                    if (f < G && opf != OP_STOP) {
                        if (opf == OP_STUCK) {
                            stuck = true;
                            going = false;
                        } else {
                            if (q == f) lreads += rd;
                            uint8_t ch;
                            if (opf == OP_S) {
                                ch = 'X'; --j; --d; --i; ++consumed; ++tcons;
                            } else if (opf == OP_I) {
                                ch = 'I'; --d; --i; ++consumed;
                            } else {
                                ch = 'D'; --j; --d; ++tcons;
                            }
                            if (q == 0) ops[nops] = ch;
                            ++nops;
                            ++wcost;
                        }
                    }
                }
            }
            // entry_writes / words_allocated of this window in closed form
            // (stored columns per level, dptable.py:62-82, 156-171)
            unsigned wr = 0;
            if (tbg && !stuck) {
                for (int dd = q; dd <= d_min; dd += G) {
                    int ss = n - budget - (K - dd) - 1;
                    ss = ss > 1 ? ss : 1;
                    const int cnt = n - ss + 1;
                    wr += cnt > 0 ? (unsigned)cnt : 0u;
                }
            }
            wr = group_sum<G>(wr);
            lreads = group_sum<G>(lreads);
            if (tbg) {
                if (stuck) {
                    write_result(3, widx);
                    phase = NEED_PAIR;
                } else {
                    if (q == 0) {
                        dists[widx] = (uint8_t)d_min;
                        rows += d_min + 1;
                        cost += wcost;
                        reads += lreads;
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

template <int NW, int G, int LPL>
static cudaError_t launch_t(const KernelParams& base, int block, int num_sms, cudaStream_t stream,
                            uint32_t** overflow, size_t* overflow_cap, LaunchShape* shape) {
    using GE = Geo<NW>;
    KernelParams P = base;
    if (block < G || block > kMaxBlock || block % 32) block = G >= 16 ? 64 : 32;
    const int groups_per_block = block / G;
    const int smem =
        (2 * smem_pad<NW, G>() + groups_per_block * (2 * GE::WMAX * NW + GE::WMAX / 2)) * 4;
    auto kern = genasm_kernel<NW, G, LPL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    // resident warps bound the band tables' L2 footprint (≈34 KB per warp at W=64,
    // G=4); measured best on config 3 with occupancy-limited residency (≈24 warps)
    const char* cap_env = getenv("GA_WARPS_PER_SM");
    const int warps_cap = cap_env && atoi(cap_env) > 0 ? atoi(cap_env) : 64;
    const int bcap = warps_cap * 32 / block;
    if (bcap >= 1 && per_sm > bcap) per_sm = bcap;
    int grid = num_sms * per_sm;
    const int64_t max_useful = (P.n_pairs + groups_per_block - 1) / groups_per_block;
    if (grid > max_useful) grid = (int)(max_useful > 0 ? max_useful : 1);
    const int levels_cap = ((P.k + 1 + G * LPL - 1) / (G * LPL)) * (G * LPL);
    P.overflow_words_per_group = GE::BAND ? (int64_t)levels_cap * P.W * NW : 0;
    constexpr int SMAX = GE::WMAX + G - 1;
    constexpr int NPASS = GE::BAND ? 1 : (GE::LV + G * LPL - 1) / (G * LPL);
    const size_t slabs = (size_t)grid * groups_per_block * (size_t)P.overflow_words_per_group;
    const size_t bands = (size_t)grid * (block / 32) * NPASS * SMAX * 32 * LPL;
    const size_t need = slabs + bands + 64;
    if (need > *overflow_cap || !*overflow) {
        if (*overflow) cudaFree(*overflow);
        *overflow = nullptr;
        *overflow_cap = 0;
        e = cudaMalloc(overflow, need * 4 + 64);
        if (e != cudaSuccess) return e;
        *overflow_cap = need;
    }
    P.overflow = *overflow;
    P.band = *overflow + ((slabs + 63) & ~(size_t)63);  // 256-byte aligned band region
    kern<<<grid, block, smem, stream>>>(P);
    shape->grid = grid;
    shape->block = block;
    shape->smem_bytes = smem;
    shape->group = G;
    shape->blocks_per_sm = per_sm;
    shape->overflow_words_per_group = P.overflow_words_per_group;
    shape->launches = 1;
    return cudaGetLastError();
}

template <int NW>
static cudaError_t launch_nw(const KernelParams& P, int group, int block, int num_sms,
                             cudaStream_t stream, uint32_t** overflow, size_t* cap,
                             LaunchShape* shape) {
    switch (group) {
        // G lanes x 16/G levels per lane: 16 levels per pass
        case 4: return launch_t<NW, 4, 4>(P, block, num_sms, stream, overflow, cap, shape);
        case 8: return launch_t<NW, 8, 2>(P, block, num_sms, stream, overflow, cap, shape);
        case 16: return launch_t<NW, 16, 1>(P, block, num_sms, stream, overflow, cap, shape);

        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_genasm_lockstep(const KernelParams& P, int group, int block, int num_sms,
                          cudaStream_t stream, uint32_t** overflow, size_t* cap,
                          LaunchShape* shape) {
    if (P.W <= 32) return launch_nw<1>(P, group, block, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_nw<2>(P, group, block, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_nw<4>(P, group, block, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm
