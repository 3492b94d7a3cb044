// pack_host.cpp -- the vector inner loop of ga_pack2 (genasm_pack.cu): one
// code byte per symbol -> 2 bits per symbol (symbol x in bits 2(x%4).. of
// byte x/4), counting the symbols outside ACGT (code > 3).  Kept out of the
// .cu files so the host compiler sees the AVX2 intrinsics directly; chosen at
// run time (scalar path in genasm_pack.cu otherwise).
#include <immintrin.h>
#include <stdint.h>

namespace genasm {

bool host_has_avx2() { return __builtin_cpu_supports("avx2"); }

// Packs 32 * nblk symbols from `codes` into 8 * nblk bytes at `out`; returns
// how many of them are > 3.  Per 32 symbols: AND 3, two multiply-adds fold
// four 2-bit fields into one byte per 32-bit lane, a shuffle + permute
// gather the eight bytes.
__attribute__((target("avx2"))) int64_t pack2_avx2(const uint8_t* codes, int64_t nblk,
                                                  uint8_t* out) {
    const __m256i three = _mm256_set1_epi8(3);
    const __m256i w01 = _mm256_set1_epi16(0x0401);       // a0 + 4 a1 per 16-bit lane
    const __m256i w23 = _mm256_set1_epi32(0x00100001);   // lo + 16 hi per 32-bit lane
    const __m256i gather = _mm256_setr_epi8(0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                            -1, -1, 0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1,
                                            -1, -1, -1, -1);
    const __m256i lanes = _mm256_setr_epi32(0, 4, 1, 1, 1, 1, 1, 1);
    int64_t bad = 0;
    for (int64_t k = 0; k < nblk; ++k) {
        const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(codes + 32 * k));
        const unsigned ok = (unsigned)_mm256_movemask_epi8(
            _mm256_cmpeq_epi8(_mm256_max_epu8(v, three), three));
        bad += __builtin_popcount(~ok);
        const __m256i a = _mm256_and_si256(v, three);
        const __m256i m = _mm256_madd_epi16(_mm256_maddubs_epi16(a, w01), w23);
        const __m256i g = _mm256_permutevar8x32_epi32(_mm256_shuffle_epi8(m, gather), lanes);
        _mm_storel_epi64(reinterpret_cast<__m128i*>(out + 8 * k), _mm256_castsi256_si128(g));
    }
    return bad;
}

}  // namespace genasm
