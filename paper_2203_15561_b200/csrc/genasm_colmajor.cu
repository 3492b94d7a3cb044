// genasm_colmajor.cu -- thread-per-window fused GenASM-DC + GenASM-TB (sm_100a).
//
// Every LANE owns one pair and walks its window chain (pkg/src/bitalign/
// window.py:95-120); the 32 lanes of a warp advance in lock-step rounds.
//
//   DC (distance.py:97-150), column-major: a pass keeps 16 consecutive levels
//     R[16p .. 16p+15][j] of the current column in registers (NW words each)
//     and sweeps the text columns j = 1..n once, evaluating the recurrence
//     level by level inside the column:
//         R[d][j] = (sh(R[d][j-1]) | PM[T[j-1]]) & sh(R[d-1][j-1] & R[d-1][j]) & R[d-1][j-1]
//     No shuffles, no wavefront fill/drain, every lane busy on its own window:
//     10 logic/shift ops per 64-bit entry plus one funnel shift for the band.
//     Early termination (key idea 2) at pass granularity: the window's DC ends
//     with the first pass whose column-n rows hold a level with bit m-1 clear.
//   Table (key ideas 1, 3): one status row per entry, and only the 32-bit band
//     around the diagonal the traceback can reach (see genasm_kernel.cuh for
//     the proof that the band holds every bit TB reads when d_min <= 15).  The
//     band words go to a per-warp global region laid out lane-interleaved
//     ([level][column pair][lane] x uint2), so each store instruction of the
//     warp writes 256 contiguous bytes.  A window that needs level 16 restarts
//     in full mode (full-width rows, [level][column][lane][NW]).
//   TB (backtrace.py:113-160): each lane walks its own window's table; the
//     match-first fast path evaluates four diagonal states per round with
//     independent loads.
#include "genasm_device.cuh"

namespace genasm {

namespace {

constexpr int kLVP = 16;           // levels per pass (registers)
constexpr int kCmBlock = 256;      // threads per block

template <int NW>
struct CmGeo {
    static constexpr int WMAX = 32 * NW;
    static constexpr bool BAND = NW >= 2;
    static constexpr int LVT = BAND ? 16 : 48;  // levels in the band/row table
    static constexpr int BAND_MAX = 32 * NW - 32;
    static constexpr int64_t TAB_WORDS = (int64_t)LVT * WMAX * 32;   // per warp
    static constexpr int CHUNK_WORDS = WMAX / 4 * 32;                // per warp, one chunk
};

// lane-interleaved chunk bytes in shared memory: byte x of this lane's chunk
__device__ __forceinline__ int chunk_byte(const uint32_t* base, int lane, int x) {
    return (int)((base[(x >> 2) * 32 + lane] >> (8 * (x & 3))) & 0xFFu);
}

template <int NW>
__global__ void __launch_bounds__(kCmBlock)
genasm_colmajor_kernel(const KernelParams P, const int64_t warp_words) {
    using CG = CmGeo<NW>;
    constexpr int WMAX = CG::WMAX;
    constexpr bool BAND = CG::BAND;
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    uint32_t* pchunk = smem + warp * 2 * CG::CHUNK_WORDS;  // forward pattern chunk
    uint32_t* tchunk = pchunk + CG::CHUNK_WORDS;           // forward text chunk
    // per-warp global region: band/row table | full-mode slab | carry row
    uint32_t* wreg = P.overflow + gw * warp_words;
    uint2* band2 = reinterpret_cast<uint2*>(wreg);
    uint32_t* band1 = wreg;
    const int W = P.W, O = P.O, K = P.k;
    const int flv = ((K + 1 + kLVP - 1) / kLVP) * kLVP;
    uint32_t* fslab = wreg + CG::TAB_WORDS;
    uint32_t* carry = fslab + (BAND ? (int64_t)flv * WMAX * 32 * NW : 0);
    PairResult* results = reinterpret_cast<PairResult*>(P.results);
    const uint32_t lut_lo = (uint32_t)P.prio_lut, lut_hi = (uint32_t)(P.prio_lut >> 32);
    const bool mfirst = ((P.prio_lut >> 60) & 0xFu) == OP_M;

    // ---- lane state ----
    int phase = NEED_PAIR;
    int64_t pair = 0, p = 0, t = 0, nops = 0;
    int Lp = 0, Lt = 0, widx = 0, m = 1, n = 0, budget = 0, pass = 0, d_min = 0;
    bool full = false;
    const uint8_t* Pp = nullptr;
    const uint8_t* Tp = nullptr;
    uint8_t* ops = nullptr;
    uint8_t* dists = nullptr;
    int64_t cost = 0, rows = 0, reads = 0, writes = 0, words = 0;
    uint32_t PM[4][NW];

    auto finish = [&](int status) {
        PairResult r{};
        r.status = status;
        r.fail_window = (status == 1 || status == 3) ? widx : -1;
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

    // copy `len` bytes from global `src` into this lane's interleaved chunk
    auto stage = [&](uint32_t* dst, const uint8_t* src, int len) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(src);
        const uint32_t* w0 = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
        const int sh = (int)(a & 3) * 8;
        const int nw = (len + 3) >> 2;
        for (int x = 0; x < nw; ++x) {
            // aligned words only; the high word is read only if it holds chunk bytes
            const uint32_t lo = w0[x];
            const uint32_t hi = (sh && 4 * (x + 1) < len + (int)(a & 3)) ? w0[x + 1] : 0u;
            dst[x * 32 + lane] = sh ? __funnelshift_r(lo, hi, sh) : lo;
        }
    };

    for (;;) {
        // ============ refill: next pair for lanes that finished theirs ============
        while (phase == NEED_PAIR) {
            const unsigned long long idx = atomicAdd(P.queue, 1ull);
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
            if (Lp <= 0) finish(2);  // EmptyPattern (window.py:87-88)
            else phase = NEED_WINDOW;
        }
        // ============ window setup: geometry, chunks, pattern masks ============
        if (phase == NEED_WINDOW) {
            const int64_t remaining = Lp - p;
            const bool final_w = remaining <= W;
            m = final_w ? (int)remaining : W;
            const int64_t tleft = Lt - t;
            n = tleft < W ? (int)(tleft > 0 ? tleft : 0) : W;
            budget = final_w ? m : W - O;
            stage(pchunk, Pp + p, m);
            stage(tchunk, Tp + t, n);
            // PM[c] bit i = 0 iff reversed-chunk pattern[i] == c (distance.py:70-79)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int w = 0; w < NW; ++w) PM[c][w] = 0xffffffffu;
            for (int i = 0; i < m; ++i) {
                const int code = chunk_byte(pchunk, lane, m - 1 - i);
                const uint32_t bit = 1u << (i & 31);
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const uint32_t clr = ((i >> 5) == w) ? bit : 0u;
                    PM[0][w] &= code == 0 ? ~clr : 0xffffffffu;
                    PM[1][w] &= code == 1 ? ~clr : 0xffffffffu;
                    PM[2][w] &= code == 2 ? ~clr : 0xffffffffu;
                    PM[3][w] &= code == 3 ? ~clr : 0xffffffffu;
                }
            }
            pass = 0;
            full = false;
            if (n == 0) {  // R[d][0] = init(m, d) solves iff d >= m
                if (m <= K) {
                    d_min = m;
                    phase = IN_TB;
                } else {
                    finish(1);
                    phase = NEED_PAIR;
                }
            } else {
                phase = IN_DC;
            }
        }
        if (__all_sync(FULL, phase == DONE)) break;
        __syncwarp();

        // ============ DC pass: 16 levels, column-major, every lane on its window ============
        {
            const bool active = phase == IN_DC;
            const int base_d = pass * kLVP;
            uint32_t col[kLVP][NW];
#pragma unroll
            for (int k = 0; k < kLVP; ++k) init_row<NW>(col[k], m, base_d + k);
            uint32_t a0[NW];  // R[base_d-1][j-1]
            init_row<NW>(a0, m, base_d > 0 ? base_d - 1 : 0);
            const uint32_t lvl0 = base_d == 0 ? 0xffffffffu : 0u;
            const bool use_carry = active && base_d > 0;
            const bool store_full = BAND && active && full;
            const bool store_band = active && !(BAND && full);
            const bool store_carry = active && (!BAND || full);
            const int steps = __reduce_max_sync(FULL, active ? n : 0);
            const int amt0 = m - 1 - n + 1 - 15;  // band origin of column index c: amt0 + c
            int found = -1;
            uint32_t keep[kLVP];
#pragma unroll
            for (int k = 0; k < kLVP; ++k) keep[k] = 0u;
            for (int c = 0; c < steps; ++c) {
                const int tx = n - 1 - c;  // reversed text index (window.py:100)
                const int code = chunk_byte(tchunk, lane, tx > 0 ? tx : 0);
                uint32_t pm[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    uint32_t x = 0xffffffffu;
                    x = code == 0 ? PM[0][w] : x;
                    x = code == 1 ? PM[1][w] : x;
                    x = code == 2 ? PM[2][w] : x;
                    x = code == 3 ? PM[3][w] : x;
                    pm[w] = x;
                }
                // level base_d: S/D/I edges from the carry row (previous pass), none at level 0
                uint32_t b0[NW];
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    b0[w] = use_carry ? carry[((int64_t)c * 32 + lane) * NW + w] : 0xffffffffu;
                uint32_t prev_old[NW];
                {
                    uint32_t tt[NW], st[NW], sv[NW];
#pragma unroll
                    for (int w = 0; w < NW; ++w) tt[w] = a0[w] & b0[w];
                    shl1<NW>(tt, st);
                    shl1<NW>(col[0], sv);
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        prev_old[w] = col[0][w];
                        col[0][w] = (sv[w] | pm[w]) & ((st[w] & a0[w]) | lvl0);
                        a0[w] = b0[w];
                    }
                }
#pragma unroll
                for (int k = 1; k < kLVP; ++k) {
                    uint32_t tt[NW], st[NW], sv[NW];
#pragma unroll
                    for (int w = 0; w < NW; ++w) tt[w] = prev_old[w] & col[k - 1][w];
                    shl1<NW>(tt, st);
                    shl1<NW>(col[k], sv);
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        const uint32_t old = col[k][w];
                        col[k][w] = (sv[w] | pm[w]) & st[w] & prev_old[w];
                        prev_old[w] = old;
                    }
                }
                // ---- table stores ----
                int amt = amt0 + c;
                amt = amt < 0 ? 0 : (amt > CG::BAND_MAX ? CG::BAND_MAX : amt);
#pragma unroll
                for (int k = 0; k < kLVP; ++k) {
                    if (BAND) {
                        const uint32_t bw = band32<NW>(col[k], amt);
                        if (c & 1) {
                            if (store_band)
                                band2[((int64_t)k * (WMAX / 2) + (c >> 1)) * 32 + lane] =
                                    make_uint2(keep[k], bw);
                        } else {
                            keep[k] = bw;
                        }
                        if (store_full) {
                            uint32_t* dst = fslab + (((int64_t)(base_d + k) * WMAX + c) * 32 + lane) * NW;
#pragma unroll
                            for (int w = 0; w < NW; ++w) dst[w] = col[k][w];
                        }
                    } else if (store_band) {
                        band1[((int64_t)(base_d + k) * WMAX + c) * 32 + lane] = col[k][0];
                    }
                }
                if (store_carry) {
#pragma unroll
                    for (int w = 0; w < NW; ++w)
                        carry[((int64_t)c * 32 + lane) * NW + w] = col[kLVP - 1][w];
                }
                if (c == n - 1 && active) {  // column n: first level whose bit m-1 is clear
                    const int tw = (m - 1) >> 5;
                    const uint32_t tb = 1u << ((m - 1) & 31);
#pragma unroll
                    for (int k = kLVP - 1; k >= 0; --k)
                        if ((word_sel<NW>(col[k], tw) & tb) == 0u && base_d + k <= K) found = k;
                }
            }
            if (BAND && (steps & 1) && store_band) {  // last (unpaired) even column
#pragma unroll
                for (int k = 0; k < kLVP; ++k)
                    band2[((int64_t)k * (WMAX / 2) + (steps >> 1)) * 32 + lane] = make_uint2(keep[k], 0u);
            }
            if (active) {
                if (found >= 0) {
                    d_min = base_d + found;
                    phase = IN_TB;
                } else if (base_d + kLVP > K) {  // NotFound(k) -> WindowFailed(index, k)
                    finish(1);
                    phase = NEED_PAIR;
                } else if (BAND && !full) {
                    full = true;  // d_min > 15: the band cannot serve TB; redo full width
                    pass = 0;
                } else {
                    ++pass;
                }
            }
        }
        __syncwarp();

        // ============ TB: each lane walks its own window ============
        if (phase == IN_TB) {
            const int cbase = m - 1 - n - 15;  // band origin of column col: cbase + col
            int d = d_min, j = n, i = m - 1, consumed = 0, tcons = 0, wcost = 0, no = 0;
            int64_t lreads = 0;
            bool stuck = false;
            uint8_t* out = ops + nops;
            // table bit x of entry (level e, column col >= 1); 1 = inactive
            auto tbit = [&](int e, int col, int x) -> uint32_t {
                const int cc = col - 1;
                if (BAND && full) {
                    const uint32_t* row = fslab + (((int64_t)e * WMAX + cc) * 32 + lane) * NW;
                    return row[x >> 5] >> (x & 31);
                }
                if (!BAND) return band1[((int64_t)e * WMAX + cc) * 32 + lane] >> x;
                const uint2 v2 = band2[((int64_t)e * (WMAX / 2) + (cc >> 1)) * 32 + lane];
                const uint32_t word = (cc & 1) ? v2.y : v2.x;
                int a1 = cbase + col;
                a1 = a1 < 0 ? 0 : (a1 > CG::BAND_MAX ? CG::BAND_MAX : a1);
                return word >> (unsigned)(x - a1);
            };
            while (i >= 0 && consumed < budget && j > 0) {
                if (mfirst && !(BAND && full)) {
                    // match runs: four diagonal states per round, independent loads
                    for (;;) {
                        unsigned mask = 0;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int ik = i - k, colk = j - 1 - k;  // state (d, j-k, i-k)
                            const bool valid = ik >= 1 && colk >= 1 && consumed + k < budget;
                            const int cc = valid ? colk : 1;
                            const int tcode = chunk_byte(tchunk, lane, n - 1 - cc);  // ct[cc] (reversed)
                            const int pcode = chunk_byte(pchunk, lane, m - 1 - (valid ? ik : 0));
                            const uint32_t bit = tbit(d, cc, valid ? ik - 1 : 0);
                            const bool ok = valid && tcode < 4 && pcode == tcode && !(bit & 1u);
                            mask |= (unsigned)ok << k;
                        }
                        const int r = __ffs(~mask) - 1;
                        for (int k = 0; k < r; ++k) out[no + k] = '=';
                        lreads += (int64_t)r * (d > 0 ? 3 : 1);
                        no += r;
                        i -= r;
                        j -= r;
                        consumed += r;
                        tcons += r;
                        if (r < 4) break;
                    }
                    if (!(i >= 0 && consumed < budget && j > 0)) break;
                }
                // full evaluation of state (d, j, i) (backtrace.py:88-99, 134-160)
                const int col1 = j - 1;
                const int dm1 = d > 0 ? d - 1 : 0;
                const int tcode = chunk_byte(tchunk, lane, n - j);  // ct[j-1]
                const int pcode = chunk_byte(pchunk, lane, m - 1 - i);
                uint32_t mb, sb, db, ib;
                if (col1 >= 1) {
                    const int x0 = i > 0 ? i - 1 : 0;
                    mb = tbit(d, col1, x0);
                    sb = tbit(dm1, col1, x0);
                    db = tbit(dm1, col1, i);
                } else {  // column 0 is init(m, .): bit x inactive iff x >= level
                    mb = i - 1 >= d;
                    sb = i - 1 >= d - 1;
                    db = i >= d - 1;
                }
                ib = tbit(dm1, j, i > 0 ? i - 1 : 0);
                const unsigned dpos = d > 0;
                const unsigned i0 = i == 0;
                const unsigned mok = (unsigned)(tcode < 4) & (unsigned)(pcode == tcode) &
                                     (i0 | (~mb & 1u));
                const unsigned sok = dpos & (i0 | (~sb & 1u));
                const unsigned iok = dpos & (i0 | (~ib & 1u));
                const unsigned dok = dpos & (~db & 1u);
                const unsigned okm = mok | sok << 1 | iok << 2 | dok << 3;
                const unsigned op = (((okm & 8u) ? lut_hi : lut_lo) >> (4u * (okm & 7u))) & 0xFu;
                if (op > OP_D) {
                    stuck = true;
                    break;
                }
                const unsigned j2 = j >= 2;
                lreads += j2 + (dpos ? j2 + 1u : 0u);
                const int dj = (0xBu >> op) & 1u, dd = (0xEu >> op) & 1u, di = (0x7u >> op) & 1u;
                out[no++] = (uint8_t)(0x4449583Du >> (8 * op));  // "=XID"
                j -= dj;
                d -= dd;
                i -= di;
                consumed += di;
                tcons += dj;
                wcost += dd;
            }
            // column 0 with pattern and budget left: i+1 insertions (backtrace.py:122-132)
            if (!stuck && i >= 0 && consumed < budget && j == 0) {
                if (i + 1 > d) {
                    stuck = true;
                } else {
                    const int left = budget - consumed;
                    const int take = i + 1 < left ? i + 1 : left;
                    for (int u = 0; u < take; ++u) out[no + u] = 'I';
                    no += take;
                    wcost += take;
                    consumed += take;
                    i -= take;
                }
            }
            if (stuck) {
                finish(3);
                phase = NEED_PAIR;
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
                    phase = NEED_WINDOW;
                } else {
                    finish(0);
                    phase = NEED_PAIR;
                }
            }
        }
    }
}

}  // namespace

template <int NW>
static cudaError_t launch_cm_t(const KernelParams& base, int num_sms, cudaStream_t stream,
                               uint32_t** overflow, size_t* overflow_cap, LaunchShape* shape) {
    using CG = CmGeo<NW>;
    KernelParams P = base;
    const int block = kCmBlock;
    const int smem = (block / 32) * 2 * CG::CHUNK_WORDS * 4;
    auto kern = genasm_colmajor_kernel<NW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const char* env = getenv("GA_CM_BLOCKS");
    if (env && atoi(env) > 0 && atoi(env) < per_sm) per_sm = atoi(env);
    int grid = num_sms * per_sm;
    const int64_t max_useful = (P.n_pairs + block - 1) / block;
    if (grid > max_useful) grid = (int)(max_useful > 0 ? max_useful : 1);
    const int flv = ((P.k + 1 + kLVP - 1) / kLVP) * kLVP;
    const int64_t warp_words = CG::TAB_WORDS +
                               (CG::BAND ? (int64_t)flv * CG::WMAX * 32 * NW : 0) +
                               (int64_t)CG::WMAX * 32 * NW;
    const size_t need = (size_t)grid * (block / 32) * (size_t)warp_words;
    if (need > *overflow_cap || !*overflow) {
        if (*overflow) cudaFree(*overflow);
        *overflow = nullptr;
        *overflow_cap = 0;
        e = cudaMalloc(overflow, need * 4 + 256);
        if (e != cudaSuccess) return e;
        *overflow_cap = need;
    }
    P.overflow = *overflow;
    P.overflow_words_per_group = warp_words;
    kern<<<grid, block, smem, stream>>>(P, warp_words);
    shape->grid = grid;
    shape->block = block;
    shape->smem_bytes = smem;
    shape->group = 1;
    shape->blocks_per_sm = per_sm;
    shape->overflow_words_per_group = warp_words;
    return cudaGetLastError();
}

cudaError_t launch_genasm_colmajor(const KernelParams& P, int num_sms, cudaStream_t stream,
                                   uint32_t** overflow, size_t* cap, LaunchShape* shape) {
    if (P.W <= 32) return launch_cm_t<1>(P, num_sms, stream, overflow, cap, shape);
    if (P.W <= 64) return launch_cm_t<2>(P, num_sms, stream, overflow, cap, shape);
    if (P.W <= 128) return launch_cm_t<4>(P, num_sms, stream, overflow, cap, shape);
    return cudaErrorInvalidValue;
}

}  // namespace genasm
