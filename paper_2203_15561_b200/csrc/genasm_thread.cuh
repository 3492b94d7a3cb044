// genasm_thread.cuh -- one window of improved GenASM (DC + TB) computed by ONE
// thread: the building blocks of the lane-per-pair kernel (genasm_thread.cu).
// Host + device code, so tools/thread_model.cpp can check it against the
// oracle on the CPU.
//
// Reference algorithm (0 = active):
//   R[d][0] = init(m, d)              bits < min(d, m) zero  (bitvec.py:108-122)
//   R[0][j] = sh(R[0][j-1]) | PM[T[j-1]]                      (distance.py:125-133)
//   R[d][j] = (sh(R[d][j-1]) | PM) & sh(R[d-1][j-1] & R[d-1][j]) & R[d-1][j-1]
//                                                               (distance.py:134-149)
// with sh(x) = x << 1 shifting in an active 0, cp / ct the reversed chunks
// (window.py:99-100) and success at bit m-1 of R[d][n].
//
// Diagonal band (fast tier, d_min <= 15).  Cell (i, j) lies on diagonal
// offset delta = (m-1-i) - (n-j).  An active cell at |delta'| >= 16 can only
// reach offset delta by |delta'| - |delta| insertion/deletion edges, each one
// level up, so it can influence level d only if |delta| >= 16 - d.  Every
// cell the traceback reads from a window with d_min <= 15 has
// |delta| <= d_min - d <= 15 - d (and its predecessors at level d-1 have
// |delta +- 1| <= 15 - (d-1)), and the success cell has delta = 0: all are
// exact when each row is kept only on the 32 diagonals delta in [-16, 15],
// everything outside treated as inactive.  Column j keeps bits
// [o_j, o_j + 31], o_j = m - n + j - 16 (bits below 0 are virtual and stay
// active, as the zeros sh() shifts in).  Moving one column right the band
// moves up one bit, so in band coordinates
//   M: sh(R[d][j-1])   -> R[d][j-1] unchanged      S: sh(R[d-1][j-1]) -> a
//   I: sh(R[d-1][j])   -> (b << 1) | f            D: R[d-1][j-1]     -> (a >> 1) | 2^31
// (a = R[d-1][j-1], b = R[d-1][j]; the filled bits are out-of-band cells,
// f = 0 while the bit below the band is virtual).  Four 32-bit operations
// per entry instead of 5 * ceil(m/32).
//
// Full tier (d_min > 15): full-width 64-bit rows, 4 levels per pass, rows
// kept in a per-lane table for the traceback.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define GA_HD __host__ __device__ __forceinline__
#else
#define GA_HD inline
#endif

namespace genasm {
namespace thr {

constexpr int kFastLevels = 16;   // levels of the band tier (d_min <= 15)
constexpr int kPassLevels = 4;    // levels per pass of the full tier

enum : int { OPC_M = 0, OPC_S = 1, OPC_I = 2, OPC_D = 3, OPC_STUCK = 5 };

// 2-bit planes of up to 64 symbols, REVERSED: bit x describes src[len-1-x].
// b0/b1 = bits 0/1 of the code, bn = code 4 (no mask: never matches).
struct Planes {
    uint64_t b0, b1, bn;
};

GA_HD uint64_t brev64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __brevll(x);
#else
    x = ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
    x = ((x >> 2) & 0x3333333333333333ull) | ((x & 0x3333333333333333ull) << 2);
    x = ((x >> 4) & 0x0F0F0F0F0F0F0F0Full) | ((x & 0x0F0F0F0F0F0F0F0Full) << 4);
    x = ((x >> 8) & 0x00FF00FF00FF00FFull) | ((x & 0x00FF00FF00FF00FFull) << 8);
    x = ((x >> 16) & 0x0000FFFF0000FFFFull) | ((x & 0x0000FFFF0000FFFFull) << 16);
    return (x >> 32) | (x << 32);
#endif
}

// four code bytes -> the nibble of one bit plane (byte k -> bit k)
GA_HD uint32_t nib(uint32_t w, int bit) {
    return (((w >> bit) & 0x01010101u) * 0x01020408u) >> 24;
}

// planes of src[0..len), 1 <= len <= 64, reversed
GA_HD Planes load_planes(const uint8_t* src, int len) {
    uint64_t f0 = 0, f1 = 0, fn = 0;
#ifdef __CUDA_ARCH__
    // aligned 4-byte words covering [src, src+len); a word never crosses the
    // allocation because allocations are at least 4-byte granular
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const int sh = (int)(a & 3);  // bytes of the first word before src
    const int nw = (sh + len + 3) >> 2;
    for (int k = 0; k < nw; ++k) {
        const uint32_t w = __ldg(wp + k);
        const int pos = 4 * k - sh;  // symbol index of the word's byte 0
        const uint64_t n0 = nib(w, 0), n1 = nib(w, 1), nn = nib(w, 2);
        if (pos >= 0) {
            f0 |= n0 << pos;
            f1 |= n1 << pos;
            fn |= nn << pos;
        } else {
            f0 |= n0 >> -pos;
            f1 |= n1 >> -pos;
            fn |= nn >> -pos;
        }
    }
#else
    for (int k = 0; k < len; ++k) {
        f0 |= (uint64_t)(src[k] & 1) << k;
        f1 |= (uint64_t)((src[k] >> 1) & 1) << k;
        fn |= (uint64_t)((src[k] >> 2) & 1) << k;
    }
#endif
    const int s = 64 - len;  // reverse the first len bits
    Planes p;
    p.b0 = brev64(f0) >> s;
    p.b1 = brev64(f1) >> s;
    p.bn = brev64(fn) >> s;
    return p;
}

// planes of symbols [start, start+len), 1 <= len <= 64, from the bit-plane
// form of the codes (bit x of word x/64 of each plane), reversed
GA_HD Planes load_planes_bits(const uint64_t* pl, int64_t plane_words, int64_t start, int len) {
    const int64_t wi = start >> 6;
    const int r = (int)(start & 63);
    uint64_t f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint64_t* q = pl + k * plane_words + wi;
#ifdef __CUDA_ARCH__
        const uint64_t w0 = __ldg(q), w1 = __ldg(q + 1);
#else
        const uint64_t w0 = q[0], w1 = q[1];
#endif
        f[k] = r ? (w0 >> r) | (w1 << (64 - r)) : w0;
    }
    const int s = 64 - len;
    Planes p;
    p.b0 = brev64(f[0]) >> s;
    p.b1 = brev64(f[1]) >> s;
    p.bn = brev64(f[2]) >> s;
    return p;
}

GA_HD uint32_t bit64(uint64_t x, int k) { return (uint32_t)(x >> k) & 1u; }

// all-ones iff bit k of x
GA_HD uint32_t bcast(uint64_t x, int k) { return 0u - (uint32_t)((x >> k) & 1u); }

// init(m, d) restricted to the band at origin org: band bit b is absolute org+b
GA_HD uint32_t init_band(int m, int d, int org) {
    const int z = (d < m ? d : m) - org;  // zero below band bit z
    if (z <= 0) return 0xffffffffu;
    if (z >= 32) return 0u;
    return ~((1u << z) - 1u);
}

GA_HD uint64_t init_row64(int m, int d) {
    const int z = d < m ? d : m;
    return z >= 64 ? 0ull : ~((1ull << z) - 1ull);
}

// three-input logic ops that must stay single instructions
GA_HD uint32_t and3(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
#else
    return a & b & c;
#endif
}
// (a | b) & c
GA_HD uint32_t orand(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xA8;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
#else
    return (a | b) & c;
#endif
}
// (a >> 1) | 2^31 -- the D edge in band coordinates
GA_HD uint32_t shr1_fill(uint32_t a) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(a, 1u, 1);
#else
    return (a >> 1) | 0x80000000u;
#endif
}
// bit `pos` of w; positions outside [0, 32) read as 1 (inactive)
GA_HD uint32_t wbit(uint32_t w, int pos) {
#ifdef __CUDA_ARCH__
    return __funnelshift_rc(w, 0xffffffffu, (unsigned)pos) & 1u;
#else
    return ((unsigned)pos < 32u) ? (w >> pos) & 1u : 1u;
#endif
}

// mismatch word of text symbol k (bits k of the text planes) against the
// pattern planes' 32-bit window (p0, p1, pn): bit b = 1 iff they differ
GA_HD uint32_t pm_word(uint32_t p0, uint32_t p1, uint32_t pn, const Planes& tp, int k) {
    return (p0 ^ bcast(tp.b0, k)) | (p1 ^ bcast(tp.b1, k)) | pn | bcast(tp.bn, k);
}

// Level pairing.  Reading level e at a band-tier window touches only the
// diagonals |delta| <= 15 - e, i.e. band bits [e, 30-e]: 31-2e bits for level
// e and 2e+1 bits for level 15-e, 32 together.  Rotated by 16, level 15-e's
// bits [15-e, 15+e] land exactly on the bits level e leaves free, so word k
// of a stored column holds levels k and 15-k (k = 0..7).
GA_HD uint32_t rot16(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __byte_perm(x, 0, 0x1032);
#else
    return (x >> 16) | (x << 16);
#endif
}
GA_HD uint32_t pair_word(uint32_t lo, uint32_t hi, int k) {
    const uint32_t mk = ((1u << (31 - 2 * k)) - 1u) << k;  // bits [k, 30-k]
    return (lo & mk) | (rot16(hi) & ~mk);
}
// stored bit at band position b of level e (0 <= e <= 15) from a column's words
GA_HD uint32_t packed_bit(uint32_t w_lo_or_hi, int e, int b) {
    const int pos = e <= 7 ? b : b + 16;
    return (w_lo_or_hi >> (pos & 31)) & 1u;
}
GA_HD int packed_word(int e) { return e <= 7 ? e : 15 - e; }

// (b << 1) | f in one instruction (LEA)
GA_HD uint32_t shl1_or(uint32_t b, uint32_t f) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 2, %2;" : "=r"(r) : "r"(b), "r"(f));
    return r;
#else
    return (b << 1) | f;
#endif
}

// Band tier DC over columns 1..n of a window (m, n >= 1), every column in its
// virtual band [o_j, o_j + 31]: band bits below absolute bit 0 are virtual
// and stay 0 (active), exactly the zeros sh() shifts in, so one recurrence
// serves every column -- only the I-edge fill differs (the bit below the band
// is virtual, 0, while o_j <= 0 and an out-of-band 1 after) and the mismatch
// word is masked to real bits.  col[] ends as R[d][n]; tab.put(j, w) receives
// each column's 8 paired words -- from column jstore on: the traceback of a
// window with d_min <= 15 never reads a column below n - budget - 15 (it
// consumes at most budget-1 pattern and d_min deletion steps before its last
// step).  Returns the mask of levels d <= 15 with R[d][n] bit m-1 active.
// one-bit rotations: the D and I edges of levels >= 1 (see dc_band)
GA_HD uint32_t rotr1(uint32_t a) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(a, a, 1);
#else
    return (a >> 1) | (a << 31);
#endif
}
GA_HD uint32_t rotl1(uint32_t b) {
#ifdef __CUDA_ARCH__
    return __funnelshift_l(b, b, 1);
#else
    return (b << 1) | (b >> 31);
#endif
}

// one band-tier column: levels 0..7 in band coordinates, levels 8..15 rotated
// by 16 (r7 carries R[7][j-1] rotated); w[] receives the 8 paired words
GA_HD void band_column(uint32_t* col, uint32_t& r7, uint32_t pm, uint32_t* w) {
    uint32_t a = col[0];
    uint32_t b = a | pm;  // level 0: the match edge only
    col[0] = b;
#pragma unroll
    for (int d = 1; d < 8; ++d) {
        const uint32_t c = col[d];
        const uint32_t nc = and3(orand(c, pm, a), rotr1(a), rotl1(b));
        a = c;
        col[d] = nc;
        b = nc;
    }
    const uint32_t pmr = rot16(pm);
    a = r7;
    b = rot16(b);
    r7 = b;
#pragma unroll
    for (int d = 8; d < kFastLevels; ++d) {
        const uint32_t c = col[d];
        const uint32_t nc = and3(orand(c, pmr, a), rotr1(a), rotl1(b));
        a = c;
        col[d] = nc;
        b = nc;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t mk = ((1u << (31 - 2 * k)) - 1u) << k;  // bits [k, 30-k]
        w[k] = (col[k] & mk) | (col[15 - k] & ~mk);
    }
}

// Band tier DC over columns 1..n of a window (m, n >= 1), every column in its
// virtual band [o_j, o_j + 31]; band bits below absolute bit 0 are virtual
// rows, active (0) like the zeros sh() shifts in: the mismatch word is masked
// to real bits.  In band coordinates R[d][j] bit x depends on R[d][j-1] bit x
// and R[d-1] bits x-1 (column j), x and x+1 (column j-1), so the bits a
// traceback of a d_min <= 15 window can read -- level e's bits [e, 30-e] --
// depend only on the same ranges one level down: every other bit may hold
// anything.  Hence the D/I shifts are plain rotations (what wraps lands on bit
// 0 or 31, outside every level >= 1's range), and levels 8..15 run rotated by
// 16 -- the position their bits take in the paired words -- so pairing is one
// LOP3 per word.  col[] ends as R[d][n]; tab.put(j, w) receives each column's
// 8 paired words from column jstore on: the traceback of a window with
// d_min <= 15 never reads a column below n - budget - 15 (it consumes at most
// budget-1 pattern and d_min deletion steps before its last step).  Returns
// the mask of levels d <= 15 with R[d][n] bit m-1 (band bit 15) active.
template <class Tab>
GA_HD uint32_t dc_band(const Planes& pp, const Planes& tp, int m, int n, int jstore, Tab& tab) {
    uint32_t col[kFastLevels];
    const int o0 = m - n - 16;
#pragma unroll
    for (int d = 0; d < kFastLevels; ++d) {
        const uint32_t v = init_band(m, d, o0);
        col[d] = d < 8 ? v : rot16(v);
    }
    uint32_t r7 = rot16(col[7]);
    uint32_t w[8];
    // columns with o_j <= 0: the band reaches below bit 0
    int jA = -o0;
    jA = jA < 0 ? 0 : (jA > n ? n : jA);
    for (int j = 1; j <= jA; ++j) {
        const int sh = -(o0 + j);  // virtual bits at the bottom of the band
        const uint32_t valid = sh < 32 ? ~0u << sh : 0u;
        const uint32_t pm = pm_word((uint32_t)(pp.b0 << sh), (uint32_t)(pp.b1 << sh),
                                    (uint32_t)(pp.bn << sh), tp, j - 1) & valid;
        band_column(col, r7, pm, w);
        if (j >= jstore) tab.put(j, w);
    }
#pragma unroll 1
    for (int j = jA + 1; j <= n; ++j) {
        const int oj = o0 + j;
        const uint32_t pm = pm_word((uint32_t)(pp.b0 >> oj), (uint32_t)(pp.b1 >> oj),
                                    (uint32_t)(pp.bn >> oj), tp, j - 1);
        band_column(col, r7, pm, w);
        if (j >= jstore) tab.put(j, w);
    }
    uint32_t ok = 0;
#pragma unroll
    for (int d = 0; d < kFastLevels; ++d) ok |= ((~col[d] >> (d < 8 ? 15 : 31)) & 1u) << d;
    return ok;
}

// (hi:lo) << 1, the high word of a 64-bit row shift
GA_HD uint32_t shl1_hi(uint32_t lo, uint32_t hi) {
#ifdef __CUDA_ARCH__
    return __funnelshift_l(lo, hi, 1);
#else
    return (hi << 1) | (lo >> 31);
#endif
}

// Full tier DC: full-width rows (two 32-bit words, W <= 64), passes of
// kPassLevels levels; every column's rows go to `ht` (column-major:
// ht.put4(d0, j, lo, hi) stores levels d0..d0+3 of column j) for the
// traceback and for the next pass.  Returns d_min <= K or -1.
template <class HTab>
GA_HD int dc_full(const Planes& pp, const Planes& tp, int m, int n, int K, HTab& ht) {
    const uint32_t p0l = (uint32_t)pp.b0, p0h = (uint32_t)(pp.b0 >> 32);
    const uint32_t p1l = (uint32_t)pp.b1, p1h = (uint32_t)(pp.b1 >> 32);
    const uint32_t pnl = (uint32_t)pp.bn, pnh = (uint32_t)(pp.bn >> 32);
    const bool thi = m - 1 >= 32;
    const uint32_t tbit = 1u << ((m - 1) & 31);
    for (int d0 = 0; d0 <= K; d0 += kPassLevels) {
        uint32_t cl[kPassLevels], ch[kPassLevels];
#pragma unroll
        for (int k = 0; k < kPassLevels; ++k) {
            const uint64_t r = init_row64(m, d0 + k);
            cl[k] = (uint32_t)r;
            ch[k] = (uint32_t)(r >> 32);
        }
        const uint64_t a0 = d0 > 0 ? init_row64(m, d0 - 1) : 0ull;
        uint32_t apl = (uint32_t)a0, aph = (uint32_t)(a0 >> 32);  // R[d0-1][j-1]
        // rows of level d0-1 (previous pass), loaded two columns ahead
        uint64_t bl1 = d0 > 0 ? ht.get(d0 - 1, 1) : 0ull;
        uint64_t bl2 = (d0 > 0 && n >= 2) ? ht.get(d0 - 1, 2) : 0ull;
        for (int j = 1; j <= n; ++j) {
            const uint64_t bcur = bl1;
            bl1 = bl2;
            bl2 = (d0 > 0 && j + 2 <= n) ? ht.get(d0 - 1, j + 2) : 0ull;
            const uint32_t s0 = bcast(tp.b0, j - 1), s1 = bcast(tp.b1, j - 1),
                           sn = bcast(tp.bn, j - 1);
            const uint32_t pml = (p0l ^ s0) | (p1l ^ s1) | pnl | sn;
            const uint32_t pmh = (p0h ^ s0) | (p1h ^ s1) | pnh | sn;
            uint32_t al = apl, ah = aph;                      // R[d-1][j-1]
            uint32_t xal = al << 1, xah = shl1_hi(al, ah);    // sh(R[d-1][j-1])
            uint32_t bl = (uint32_t)bcur, bh = (uint32_t)(bcur >> 32);  // R[d-1][j]
#pragma unroll
            for (int k = 0; k < kPassLevels; ++k) {
                const uint32_t xl = cl[k] << 1, xh = shl1_hi(cl[k], ch[k]);
                uint32_t nl, nh;
                if (k == 0 && d0 == 0) {  // level 0: the match edge only
                    nl = xl | pml;
                    nh = xh | pmh;
                } else {
                    nl = and3(orand(xl, pml, xal), bl << 1, al);
                    nh = and3(orand(xh, pmh, xah), shl1_hi(bl, bh), ah);
                }
                al = cl[k];
                ah = ch[k];
                xal = xl;
                xah = xh;
                bl = nl;
                bh = nh;
                cl[k] = nl;
                ch[k] = nh;
            }
            ht.put4(d0, j, cl, ch);
            apl = (uint32_t)bcur;
            aph = (uint32_t)(bcur >> 32);
        }
#pragma unroll
        for (int k = 0; k < kPassLevels; ++k)
            if (d0 + k <= K && !((thi ? ch[k] : cl[k]) & tbit)) return d0 + k;
    }
    return -1;
}

template <class HTab>
GA_HD uint32_t full_bit(HTab& ht, int e, int c, int x) {
    return (uint32_t)(ht.get(e, c) >> x) & 1u;
}

GA_HD unsigned ctz32(unsigned x) {  // count trailing zeros, x != 0
#ifdef __CUDA_ARCH__
    return __ffs(x) - 1;
#else
    return __builtin_ctz(x);
#endif
}

// symbol equality along a diagonal: bit x = (cp[x + s] == ct[x]), both in ACGT
GA_HD uint64_t diag_eq(const Planes& pp, const Planes& tp, int s) {
    uint64_t a0, a1, an;
    if (s >= 0) {
        a0 = s < 64 ? pp.b0 >> s : 0ull;
        a1 = s < 64 ? pp.b1 >> s : 0ull;
        an = s < 64 ? pp.bn >> s : ~0ull;
    } else {
        a0 = -s < 64 ? pp.b0 << -s : 0ull;
        a1 = -s < 64 ? pp.b1 << -s : 0ull;
        an = -s < 64 ? pp.bn << -s : ~0ull;
    }
    return ~((a0 ^ tp.b0) | (a1 ^ tp.b1) | an | tp.bn);
}

#ifndef GA_KRUN
#define GA_KRUN 8
#endif
constexpr int kRun = GA_KRUN;  // '=' steps speculated per round trip

// Traceback of one window (backtrace.py:88-160), from (j=n, d=d_min, i=m-1)
// until the budget is consumed.  BIT(e, c, x) returns table bit x of level e,
// column c >= 1 (1 = inactive); column 0 is init(m, .) and read analytically.
// Writes ops (ASCII) at ops[nops..]; returns false if the walk got stuck.
struct TbOut {
    int consumed, tcons, wcost;
    int64_t reads;
};

template <class BitFn>
GA_HD bool traceback(BitFn&& BIT, const Planes& pp, const Planes& tp, int m, int n, int d_min,
                     int budget, uint64_t prio_lut, uint8_t* ops, int64_t& nops, TbOut& o) {
    int d = d_min, j = n, i = m - 1;
    o.consumed = o.tcons = o.wcost = 0;
    o.reads = 0;
    const bool m_first = ((prio_lut >> 60) & 0xFu) == OPC_M;  // all four edges active -> M
    int s_eq = 1 << 30;
    uint64_t eqv = 0;
    for (;;) {
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
            if (i + 1 > d) return false;
            const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
            for (int u = 0; u < take; ++u) ops[nops + u] = 'I';
            nops += take;
            o.wcost += take;
            o.consumed += take;
            return true;
        }
        if (m_first && j >= 2 && i >= 1) {  // a run of '=' steps, kRun reads in flight
            int K = j - 1;
            K = K < i ? K : i;
            K = K < budget - o.consumed ? K : budget - o.consumed;
            K = K < kRun ? K : kRun;
            const int sd = i - (j - 1);
            if (sd != s_eq) {
                s_eq = sd;
                eqv = diag_eq(pp, tp, sd);
            }
            uint32_t mbk[kRun];
#pragma unroll
            for (int k = 0; k < kRun; ++k) mbk[k] = k < K ? BIT(d, j - 1 - k, i - 1 - k) : 1u;
            unsigned okm = 0;
#pragma unroll
            for (int k = 0; k < kRun; ++k)
                okm |= (((uint32_t)(eqv >> ((j - 1 - k) & 63)) & 1u) & ~mbk[k]) << k;
            okm &= (1u << K) - 1u;
            const int run = (int)ctz32(~okm);
            for (int k = 0; k < run; ++k) ops[nops + k] = '=';
            nops += run;
            j -= run;
            i -= run;
            o.consumed += run;
            o.tcons += run;
            o.reads += (int64_t)run * (d > 0 ? 3 : 1);
            if (run == K) continue;
            if (i < 0 || o.consumed >= budget) return true;
        }
        const bool symeq = !bit64(tp.bn, j - 1) && !bit64(pp.bn, i) &&
                           bit64(tp.b0, j - 1) == bit64(pp.b0, i) &&
                           bit64(tp.b1, j - 1) == bit64(pp.b1, i);
        const int dm1 = d > 0 ? d - 1 : 0;
        uint32_t mb = 0, sb = 0, db, ib = 0;
        if (j == 1) {  // column 0 = init(m, .): bit x inactive iff x >= level
            mb = i - 1 >= d;
            sb = i - 1 >= d - 1;
            db = i >= d - 1;
        } else {
            if (i >= 1) {
                mb = BIT(d, j - 1, i - 1);
                sb = BIT(dm1, j - 1, i - 1);
            }
            db = BIT(dm1, j - 1, i);
        }
        if (i >= 1) ib = BIT(dm1, j, i - 1);
        const bool dpos = d > 0;
        const bool mok = symeq && (i == 0 || !mb);
        const bool sok = dpos && (i == 0 || !sb);
        const bool iok = dpos && (i == 0 || !ib);
        const bool dok = dpos && !db;
        const unsigned okm =
            (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
        const int op = (int)((prio_lut >> (4 * okm)) & 0xFu);
        o.reads += (j >= 2) + (dpos ? (j >= 2) + 1 : 0);
        if (op == OPC_M) {
            ops[nops++] = '=';
            --j; --i; ++o.consumed; ++o.tcons;
        } else if (op == OPC_S) {
            ops[nops++] = 'X';
            --j; --d; --i; ++o.consumed; ++o.tcons; ++o.wcost;
        } else if (op == OPC_I) {
            ops[nops++] = 'I';
            --d; --i; ++o.consumed; ++o.wcost;
        } else if (op == OPC_D) {
            ops[nops++] = 'D';
            --j; --d; ++o.tcons; ++o.wcost;
        } else {
            return false;
        }
    }
}

// first table column the band-tier traceback can read (see dc_band)
GA_HD int band_jstore(int n, int budget) {
    const int j = n - budget - 15;
    return j > 1 ? j : 1;
}

// Traceback of a band-tier window: the walk of traceback() with the level
// bits read from the band table (tab.wi(e): the word of level e, tab.bit(w, e,
// b): its bit at band position b, relative to each column's virtual band
// origin o_j) and the '=' test from the symbol planes.

// kWriteEq = false: the ops buffer was pre-filled with '=', only the other ops
// are written
template <bool kWriteEq = true, class Tab>
GA_HD bool tb_band(Tab& tab, const Planes& pp, const Planes& tp, int m, int n, int d_min,
                   int budget, uint64_t prio_lut, uint8_t* ops, int64_t& nops, TbOut& o) {
    constexpr uint32_t kChars = '=' | 'X' << 8 | 'I' << 16 | 'D' << 24;
    int d = d_min, j = n, i = m - 1;
    const int o0 = m - n - 16;
    o.consumed = o.tcons = o.wcost = 0;
    o.reads = 0;
    // with '=' first in priority a step is '=' iff its match edge is active:
    // runs of them along a diagonal are found kRun at a time, their table
    // words loaded together
    const bool m_first = ((prio_lut >> 60) & 0xFu) == OPC_M;  // all four edges active -> M
    int s_eq = 1 << 30;
    uint64_t eqv = 0;
    for (;;) {
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
            if (i + 1 > d) return false;
            const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
            for (int u = 0; u < take; ++u) ops[nops + u] = 'I';
            nops += take;
            o.wcost += take;
            o.consumed += take;
            return true;
        }
        if (m_first && j >= 2 && i >= 1) {
            int K = j - 1;
            K = K < i ? K : i;
            K = K < budget - o.consumed ? K : budget - o.consumed;
            K = K < kRun ? K : kRun;
            const int sd = i - (j - 1);  // diagonal: pattern index - text index
            if (sd != s_eq) {
                s_eq = sd;
                eqv = diag_eq(pp, tp, sd);
            }
            const int u = i - (o0 + j);
            const int kd = tab.wi(d);
            const int dm1 = d > 0 ? d - 1 : 0;
            const int ke = tab.wi(dm1);
            // level d and d-1 words of columns j-1-k; level d-1 of column j too: the
            // step that ends the run reads from them as well
            uint32_t w[kRun], v[kRun];
#pragma unroll
            for (int k = 0; k < kRun; ++k) {
                w[k] = k < K ? tab.get(kd, j - 1 - k) : 0u;
                v[k] = k < K ? tab.get(ke, j - 1 - k) : 0u;
            }
            const uint32_t vj = tab.get(ke, j);
            // step k sits at (i-k, j-k): '=' iff symbols match and R[d][j-1-k] bit i-1-k
            // (band position u) is active
            unsigned okm = 0;
#pragma unroll
            for (int k = 0; k < kRun; ++k) {
                const uint32_t eq = (uint32_t)(eqv >> ((j - 1 - k) & 63)) & 1u;
                okm |= (eq & ~tab.bit(w[k], d, u)) << k;
            }
            okm &= (1u << K) - 1u;
            const int run = (int)ctz32(~okm);
            if (kWriteEq)
                for (int k = 0; k < run; ++k) ops[nops + k] = '=';
            nops += run;
            j -= run;
            i -= run;
            o.consumed += run;
            o.tcons += run;
            o.reads += (int64_t)run * (d > 0 ? 3 : 1);
            if (run == K) continue;  // limits reached: re-check at the new state
            // the step at (i, j) = run end: its '=' edge is inactive; the others
            // come from the words already loaded (j >= 2, i >= 1 here)
            uint32_t wr = v[0], wp = vj;
#pragma unroll
            for (int k = 1; k < kRun; ++k) {
                wr = run == k ? v[k] : wr;
                wp = run == k ? v[k - 1] : wp;
            }
            const bool dpos = d > 0;
            const bool sok = dpos && !tab.bit(wr, dm1, u);
            const bool iok = dpos && !tab.bit(wp, dm1, u - 1);
            const bool dok = dpos && !tab.bit(wr, dm1, u + 1);
            const unsigned om = (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
            const int op = (int)((prio_lut >> (4 * om)) & 0xFu);
            o.reads += dpos ? 3 : 1;
            if (op > OPC_D) return false;
            ops[nops++] = (uint8_t)(kChars >> (8 * op));
            const int mj = op != OPC_I, mi = op != OPC_D;
            j -= mj;
            i -= mi;
            d -= 1;
            o.consumed += mi;
            o.tcons += mj;
            o.wcost += 1;
            continue;
        }
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) continue;
        const int u = i - (o0 + j);  // band position of (i, j); (i-1, j-1) shares it
        const int dm1 = d > 0 ? d - 1 : 0;
        const uint32_t wj = tab.get(tab.wi(dm1), j);
        uint32_t mb, sb, db;
        if (j >= 2) {
            const uint32_t w1 = tab.get(tab.wi(d), j - 1);
            const uint32_t w2 = tab.get(tab.wi(dm1), j - 1);
            mb = tab.bit(w1, d, u);
            sb = tab.bit(w2, dm1, u);
            db = tab.bit(w2, dm1, u + 1);
        } else {  // column 0 = init(m, .): bit x inactive iff x >= level
            mb = i - 1 >= d;
            sb = i - 1 >= d - 1;
            db = i >= d - 1;
        }
        const uint32_t ib = tab.bit(wj, dm1, u - 1);
        const bool symeq = !bit64(tp.bn, j - 1) && !bit64(pp.bn, i) &&
                           bit64(tp.b0, j - 1) == bit64(pp.b0, i) &&
                           bit64(tp.b1, j - 1) == bit64(pp.b1, i);
        const bool dpos = d > 0;
        const bool i0 = i == 0;
        const bool mok = symeq && (i0 || !mb);
        const bool sok = dpos && (i0 || !sb);
        const bool iok = dpos && (i0 || !ib);
        const bool dok = dpos && !db;
        const unsigned okm =
            (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
        const int op = (int)((prio_lut >> (4 * okm)) & 0xFu);
        o.reads += (j >= 2) + (dpos ? (j >= 2) + 1 : 0);
        if (op > OPC_D) return false;
        if (kWriteEq || op != OPC_M) ops[nops] = (uint8_t)(kChars >> (8 * op));
        ++nops;
        const int mj = op != OPC_I;  // M, S, D consume a text symbol
        const int mi = op != OPC_D;  // M, S, I consume a pattern symbol
        const int md = op != OPC_M;
        j -= mj;
        i -= mi;
        d -= md;
        o.consumed += mi;
        o.tcons += mj;
        o.wcost += md;
    }
}

// Traceback of a band window over any table format (the band tier's and the
// wide tier's; tools/thread_model.cpp), the walk of traceback() with the level
// bits read from the table.  Tab supplies the table format:
//   Tab::Word          the stored word type (32-bit band tier, 64-bit wide tier)
//   Tab::kHalf         band half-width: column j keeps absolute pattern bits
//                      [o_j, o_j + 2 kHalf), o_j = m - n + j - kHalf
//   tab.get(e, c)      the word of column c >= 1 that holds level e
//   tab.bit(w, e, x)   level e's bit at band position x of such a word
// and the '=' test comes from the symbol planes.
//
// kWriteEq = false: the ops buffer was pre-filled with '=', only the other ops
// are written
template <bool kWriteEq = true, int kR = kRun, class Tab>
GA_HD bool tb_band_t(Tab& tab, const Planes& pp, const Planes& tp, int m, int n, int d_min,
                   int budget, uint64_t prio_lut, uint8_t* ops, int64_t& nops, TbOut& o) {
    using Word = typename Tab::Word;
    constexpr uint32_t kChars = '=' | 'X' << 8 | 'I' << 16 | 'D' << 24;
    int d = d_min, j = n, i = m - 1;
    const int o0 = m - n - Tab::kHalf;
    o.consumed = o.tcons = o.wcost = 0;
    o.reads = 0;
    // with '=' first in priority a step is '=' iff its match edge is active:
    // runs of them along a diagonal are found kR at a time, their table
    // words loaded together
    const bool m_first = ((prio_lut >> 60) & 0xFu) == OPC_M;  // all four edges active -> M
    int s_eq = 1 << 30;
    uint64_t eqv = 0;
    for (;;) {
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) {  // column 0: init zeros cover i+1 insertions at level d
            if (i + 1 > d) return false;
            const int take = (i + 1 < budget - o.consumed) ? i + 1 : budget - o.consumed;
            for (int u = 0; u < take; ++u) ops[nops + u] = 'I';
            nops += take;
            o.wcost += take;
            o.consumed += take;
            return true;
        }
        if (m_first && j >= 2 && i >= 1) {
            int K = j - 1;
            K = K < i ? K : i;
            K = K < budget - o.consumed ? K : budget - o.consumed;
            K = K < kR ? K : kR;
            const int sd = i - (j - 1);  // diagonal: pattern index - text index
            if (sd != s_eq) {
                s_eq = sd;
                eqv = diag_eq(pp, tp, sd);
            }
            const int u = i - (o0 + j);
            const int dm1 = d > 0 ? d - 1 : 0;
            // level d and d-1 words of columns j-1-k; level d-1 of column j too: the
            // step that ends the run reads from them as well
            Word w[kR], v[kR];
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                w[k] = k < K ? tab.get(d, j - 1 - k) : Word(0);
                v[k] = k < K ? tab.get(dm1, j - 1 - k) : Word(0);
            }
            const Word vj = tab.get(dm1, j);
            // step k sits at (i-k, j-k): '=' iff symbols match and R[d][j-1-k] bit i-1-k
            // (band position u) is active
            unsigned okm = 0;
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                const uint32_t eq = (uint32_t)(eqv >> ((j - 1 - k) & 63)) & 1u;
                okm |= (eq & ~tab.bit(w[k], d, u)) << k;
            }
            okm &= (1u << K) - 1u;
            const int run = (int)ctz32(~okm);
            if (kWriteEq)
                for (int k = 0; k < run; ++k) ops[nops + k] = '=';
            nops += run;
            j -= run;
            i -= run;
            o.consumed += run;
            o.tcons += run;
            o.reads += (int64_t)run * (d > 0 ? 3 : 1);
            if (run == K) continue;  // limits reached: re-check at the new state
            // the step at (i, j) = run end: its '=' edge is inactive; the others
            // come from the words already loaded (j >= 2, i >= 1 here)
            Word wr = v[0], wp = vj;
#pragma unroll
            for (int k = 1; k < kR; ++k) {
                wr = run == k ? v[k] : wr;
                wp = run == k ? v[k - 1] : wp;
            }
            const bool dpos = d > 0;
            const bool sok = dpos && !tab.bit(wr, dm1, u);
            const bool iok = dpos && !tab.bit(wp, dm1, u - 1);
            const bool dok = dpos && !tab.bit(wr, dm1, u + 1);
            const unsigned om = (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
            const int op = (int)((prio_lut >> (4 * om)) & 0xFu);
            o.reads += dpos ? 3 : 1;
            if (op > OPC_D) return false;
            ops[nops++] = (uint8_t)(kChars >> (8 * op));
            const int mj = op != OPC_I, mi = op != OPC_D;
            j -= mj;
            i -= mi;
            d -= 1;
            o.consumed += mi;
            o.tcons += mj;
            o.wcost += 1;
            continue;
        }
        if (i < 0 || o.consumed >= budget) return true;
        if (j == 0) continue;
        const int u = i - (o0 + j);  // band position of (i, j); (i-1, j-1) shares it
        const int dm1 = d > 0 ? d - 1 : 0;
        const Word wj = tab.get(dm1, j);
        uint32_t mb, sb, db;
        if (j >= 2) {
            const Word w1 = tab.get(d, j - 1);
            const Word w2 = tab.get(dm1, j - 1);
            mb = tab.bit(w1, d, u);
            sb = tab.bit(w2, dm1, u);
            db = tab.bit(w2, dm1, u + 1);
        } else {  // column 0 = init(m, .): bit x inactive iff x >= level
            mb = i - 1 >= d;
            sb = i - 1 >= d - 1;
            db = i >= d - 1;
        }
        const uint32_t ib = tab.bit(wj, dm1, u - 1);
        const bool symeq = !bit64(tp.bn, j - 1) && !bit64(pp.bn, i) &&
                           bit64(tp.b0, j - 1) == bit64(pp.b0, i) &&
                           bit64(tp.b1, j - 1) == bit64(pp.b1, i);
        const bool dpos = d > 0;
        const bool i0 = i == 0;
        const bool mok = symeq && (i0 || !mb);
        const bool sok = dpos && (i0 || !sb);
        const bool iok = dpos && (i0 || !ib);
        const bool dok = dpos && !db;
        const unsigned okm =
            (unsigned)mok | (unsigned)sok << 1 | (unsigned)iok << 2 | (unsigned)dok << 3;
        const int op = (int)((prio_lut >> (4 * okm)) & 0xFu);
        o.reads += (j >= 2) + (dpos ? (j >= 2) + 1 : 0);
        if (op > OPC_D) return false;
        if (kWriteEq || op != OPC_M) ops[nops] = (uint8_t)(kChars >> (8 * op));
        ++nops;
        const int mj = op != OPC_I;  // M, S, D consume a text symbol
        const int mi = op != OPC_D;  // M, S, I consume a pattern symbol
        const int md = op != OPC_M;
        j -= mj;
        i -= mi;
        d -= md;
        o.consumed += mi;
        o.tcons += mj;
        o.wcost += md;
    }
}

// ---------------------------------------------------------------------------
// Wide tier (16 <= d_min <= 31): the band of the band tier widened to the 64
// diagonals delta in [-32, 31] (column j keeps bits [O_j, O_j + 63],
// O_j = m - n + j - 32; band bit X <-> delta = 31 - X, success at X = 31).
// The band tier's argument with 32 for 16: a cell the traceback of a window
// with d_min <= 31 reads at level e has |delta| <= 31 - e, i.e. X in
// [e, 62 - e], and those bits depend only on the same ranges one level down,
// so the 64-bit D/I shifts are rotations as well.  Levels 0..16 are computed
// 64 bits wide (8 instructions per entry), levels 17..31 (|delta| <= 14) in
// the 32-bit sub-band X in [16, 47], rotated by 16 like the band tier's upper
// levels (4 instructions per entry); level 16 feeds them through one LOP3.
//
// Paired storage, the band tier's trick at 64 bits: level e <= 15 needs
// X in [e, 62 - e] (63 - 2e bits), level 31 - e needs X in [31 - e, 31 + e]
// (2e + 1 bits) -- rotated by 32 (the two 32-bit halves swapped) exactly the
// bits level e leaves free.  The rotated-by-16 32-bit form of level 31 - e
// has those bits at the same positions in both halves, so pair k (levels k
// and 31 - k) is two LOP3s: 16 pairs, 32 words (128 B) per column.
// ---------------------------------------------------------------------------
constexpr int kWideLevels = 32;

// low word of (hi:lo) >> 1 and of (hi:lo) << 1 >> 32
GA_HD uint32_t fsr1(uint32_t lo, uint32_t hi) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(lo, hi, 1);
#else
    return (lo >> 1) | (hi << 31);
#endif
}
GA_HD uint32_t fsl1(uint32_t lo, uint32_t hi) {  // (hi << 1) | (lo >> 31)
#ifdef __CUDA_ARCH__
    return __funnelshift_l(lo, hi, 1);
#else
    return (hi << 1) | (lo >> 31);
#endif
}
// the 32-bit sub-band X in [16, 47] of a 64-bit band row, rotated by 16
GA_HD uint32_t sub16(uint32_t lo, uint32_t hi) {
    return (lo & 0xffff0000u) | (hi & 0x0000ffffu);  // one LOP3
}

GA_HD uint64_t init_band64(int m, int d, int org) {
    const int z = (d < m ? d : m) - org;  // zero below band bit z
    if (z <= 0) return ~0ull;
    if (z >= 64) return 0ull;
    return ~((1ull << z) - 1ull);
}

GA_HD uint64_t shl64(uint64_t x, int s) { return s < 64 ? x << s : 0ull; }

// one wide-tier column: cl/ch = levels 0..16 (64-bit), r = levels 17..31
// (sub-band, rotated), r16 = level 16 of the previous column (sub-band,
// rotated); when `store`, tab.put4(j, q, w) receives the column's 32 paired
// words four at a time (so only four are live at once)
template <class Tab>
GA_HD void wide_column(uint32_t* cl, uint32_t* ch, uint32_t* r, uint32_t& r16, uint32_t pml,
                       uint32_t pmh, bool store, int j, Tab& tab) {
    uint32_t al = cl[0], ah = ch[0];
    uint32_t bl = al | pml, bh = ah | pmh;  // level 0: the match edge only
    cl[0] = bl;
    ch[0] = bh;
#pragma unroll
    for (int d = 1; d <= 16; ++d) {
        const uint32_t c_l = cl[d], c_h = ch[d];
        // D: (a >> 1), I: (b << 1), both as 64-bit rotations
        const uint32_t nl = and3(orand(c_l, pml, al), fsr1(al, ah), fsl1(bh, bl));
        const uint32_t nh = and3(orand(c_h, pmh, ah), fsr1(ah, al), fsl1(bl, bh));
        al = c_l;
        ah = c_h;
        cl[d] = nl;
        ch[d] = nh;
        bl = nl;
        bh = nh;
    }
    uint32_t b = sub16(bl, bh);
    uint32_t a = r16;
    r16 = b;
    const uint32_t pmr = sub16(pml, pmh);
#pragma unroll
    for (int d = 17; d < kWideLevels; ++d) {
        const uint32_t c = r[d - 17];
        const uint32_t nc = and3(orand(c, pmr, a), rotr1(a), rotl1(b));
        a = c;
        r[d - 17] = nc;
        b = nc;
    }
    if (!store) return;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k = 2 * q + h;
            const uint32_t s = k == 15 ? r16 : r[14 - k];  // level 31 - k
            const uint32_t mlo = 0xffffffffu << k;        // X in [k, 31]
            const uint32_t mhi = 0xffffffffu >> (k + 1);  // X in [32, 62 - k]
            w[2 * h] = (cl[k] & mlo) | (s & ~mlo);
            w[2 * h + 1] = (ch[k] & mhi) | (s & ~mhi);
        }
        tab.put4(j, q, w);
    }
}

// Wide tier DC over columns 1..n (m, n >= 1); tab.put4 receives each
// column's 32 paired words from column jstore on.  Returns the mask of levels
// d <= 31 with R[d][n] bit m-1 (band bit 31) active.
template <class Tab>
GA_HD uint32_t dc_wide(const Planes& pp, const Planes& tp, int m, int n, int jstore, Tab& tab) {
    uint32_t cl[17], ch[17], r[15];
    const int O0 = m - n - 32;
#pragma unroll
    for (int d = 0; d <= 16; ++d) {
        const uint64_t v = init_band64(m, d, O0);
        cl[d] = (uint32_t)v;
        ch[d] = (uint32_t)(v >> 32);
    }
    uint32_t r16 = sub16(cl[16], ch[16]);
#pragma unroll
    for (int d = 17; d < kWideLevels; ++d) r[d - 17] = rot16(init_band(m, d, O0 + 16));
#pragma unroll 1
    for (int j = 1; j <= n; ++j) {
        const int oj = O0 + j;
        uint64_t a0, a1, an, valid;
        if (oj < 0) {  // virtual bits below absolute bit 0: active, mismatch 0
            a0 = shl64(pp.b0, -oj);
            a1 = shl64(pp.b1, -oj);
            an = shl64(pp.bn, -oj);
            valid = shl64(~0ull, -oj);
        } else {
            a0 = pp.b0 >> oj;
            a1 = pp.b1 >> oj;
            an = pp.bn >> oj;
            valid = ~0ull;
        }
        const uint32_t s0 = bcast(tp.b0, j - 1), s1 = bcast(tp.b1, j - 1), sn = bcast(tp.bn, j - 1);
        const uint32_t pml = (((uint32_t)a0 ^ s0) | ((uint32_t)a1 ^ s1) | (uint32_t)an | sn) &
                             (uint32_t)valid;
        const uint32_t pmh = (((uint32_t)(a0 >> 32) ^ s0) | ((uint32_t)(a1 >> 32) ^ s1) |
                              (uint32_t)(an >> 32) | sn) & (uint32_t)(valid >> 32);
        wide_column(cl, ch, r, r16, pml, pmh, j >= jstore, j, tab);
    }
    uint32_t ok = 0;
#pragma unroll
    for (int d = 0; d <= 16; ++d) ok |= ((~cl[d] >> 31) & 1u) << d;
#pragma unroll
    for (int d = 17; d < kWideLevels; ++d) ok |= ((~r[d - 17] >> 31) & 1u) << d;
    return ok;
}

// first table column the wide-tier traceback can read (see band_jstore)
GA_HD int wide_jstore(int n, int budget) {
    const int j = n - budget - 31;
    return j > 1 ? j : 1;
}

// level e's pair in the wide table, and its bit at band position x of a pair
// word (levels >= 16 are stored with the halves swapped)
GA_HD int wide_pair(int e) { return e <= 15 ? e : 31 - e; }
GA_HD uint32_t wide_bit(uint64_t w, int e, int x) {
    return (uint32_t)(w >> ((e <= 15 ? x : x ^ 32) & 63)) & 1u;
}

// entry_writes of one window in closed form (dptable.py:62-82, 156-171):
// level d stores columns max(1, n - budget - (K - d) - 1) .. n
// level dd stores min(n, c0 - dd) columns, c0 = budget + K + 2 (n >= 0,
// dd <= d_min <= K): the first t = clamp(c0 - n + 1, 0, d_min + 1) levels store
// all n, the rest c0 - dd
GA_HD int64_t window_writes(int n, int budget, int K, int d_min) {
    const int64_t c0 = (int64_t)budget + K + 2;
    int64_t t = c0 - n + 1;
    t = t < 0 ? 0 : (t > d_min + 1 ? d_min + 1 : t);
    const int64_t rest = d_min + 1 - t;  // levels t..d_min
    return t * n + rest * c0 - ((int64_t)d_min * (d_min + 1) / 2 - t * (t - 1) / 2);
}

// first active edge in priority order for each 4-bit mask of active edges
// (backtrace.py:134-160); 5 = none
GA_HD uint64_t make_prio_lut(const char* prio) {
    uint64_t lut = 0;
    for (uint64_t mask = 0; mask < 16; ++mask) {
        uint64_t op = OPC_STUCK;
        for (int u = 3; u >= 0; --u) {
            const char c = prio[u];
            const uint64_t id = c == 'M' ? 0 : c == 'S' ? 1 : c == 'I' ? 2 : 3;
            if (mask & (1ull << id)) op = id;
        }
        lut |= op << (4 * mask);
    }
    return lut;
}

}  // namespace thr
}  // namespace genasm
