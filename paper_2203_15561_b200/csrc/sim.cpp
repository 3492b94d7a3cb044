// sim.cpp -- workload generator: an exact C++ port of the reference's
// i.i.d. read simulator and its CLI recipe, so the bench and parity inputs
// are the very pairs `bitalign simulate --emit-pairs` would produce, at
// C++ speed and in parallel (the Python generator takes ~6 min for config 3).
//
//   derive_seed     pkg/src/bitalign/sim.py:53-57
//   make_reference  pkg/src/bitalign/sim.py:60-65   (random.Random.choices)
//   simulate_read   pkg/src/bitalign/sim.py:68-103  (random(), choice())
//   CLI recipe      pkg/src/bitalign/cli.py:139-147, 162-169 (randrange positions)
//
// CPython's random.Random is MT19937 seeded by init_by_array over the
// 32-bit little-endian words of |seed|; random() = (a>>5, b>>6) / 2**53;
// _randbelow(n) = rejection-sampled getrandbits(n.bit_length()).
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <thread>
#include <vector>

#include "../../include/genasm_sim.h"

namespace {

struct MT {
    uint32_t mt[624];
    int mti = 625;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < 624; mti++)
            mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t* key, int len) {
        init_genrand(19650218u);
        int i = 1, j = 0;
        int k = 624 > len ? 624 : len;
        for (; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= 624) { mt[0] = mt[623]; i = 1; }
            if (j >= len) j = 0;
        }
        for (k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            i++;
            if (i >= 624) { mt[0] = mt[623]; i = 1; }
        }
        mt[0] = 0x80000000u;
    }
    // random.Random(seed) for a non-negative int seed < 2**64
    void seed_u64(uint64_t s) {
        uint32_t key[2] = {(uint32_t)s, (uint32_t)(s >> 32)};
        init_by_array(key, (s >> 32) ? 2 : 1);
    }
    uint32_t next() {
        static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
        uint32_t y;
        if (mti >= 624) {
            int kk;
            for (kk = 0; kk < 624 - 397; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < 623; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[623] = mt[396] ^ (y >> 1) ^ mag01[y & 1u];
            mti = 0;
        }
        y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= (y >> 18);
        return y;
    }
    double random() {
        uint32_t a = next() >> 5, b = next() >> 6;
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
    }
    uint64_t getrandbits(int k) {  // 1 <= k <= 64
        if (k <= 32) return next() >> (32 - k);
        uint64_t lo = next();
        uint64_t hi = next() >> (64 - k);
        return lo | (hi << 32);
    }
    uint64_t randbelow(uint64_t n) {  // n >= 1
        int k = 0;
        for (uint64_t x = n; x; x >>= 1) k++;
        uint64_t r = getrandbits(k);
        while (r >= n) r = getrandbits(k);
        return r;
    }
};

const uint64_t kMul = 6364136223846793005ull;
const uint64_t kInc = 1442695040888963407ull;

uint64_t derive(uint64_t seed, uint64_t salt) { return seed * kMul + salt + kInc; }

// simulate_read (sim.py:68-103); writes codes when out != null; returns length
int64_t sim_one(const uint8_t* ref, int64_t pos, int32_t length, double sub, double ins,
                double dele, uint64_t seed, uint8_t* out, char* ops = nullptr,
                int64_t* n_ops = nullptr) {
    MT rng;
    rng.seed_u64(derive(derive(seed, (uint64_t)pos), (uint64_t)length));
    const double sub_edge = dele + sub;
    int64_t n = 0, k = 0;  // read symbols, truth ops
    for (int64_t x = pos; x < pos + length; ++x) {
        const uint8_t base = ref[x];
        if (rng.random() < ins) {
            uint8_t c = (uint8_t)rng.randbelow(4);
            if (out) out[n] = c;
            if (ops) ops[k] = 'I';
            n++, k++;
        }
        const double draw = rng.random();
        if (draw < dele) {
            if (ops) ops[k] = 'D';
            k++;
            continue;
        }
        if (draw < sub_edge) {
            uint8_t r = (uint8_t)rng.randbelow(3);  // "ACGT".replace(base, "")[r]
            uint8_t c = r < base ? r : (uint8_t)(r + 1);
            if (out) out[n] = c;
            if (ops) ops[k] = 'X';
        } else {
            if (out) out[n] = base;
            if (ops) ops[k] = '=';
        }
        n++, k++;
    }
    if (n_ops) *n_ops = k;
    return n;
}

template <class F>
void parallel_for(int64_t count, int nthreads, F&& f) {
    if (nthreads <= 1 || count < 64) {
        for (int64_t q = 0; q < count; ++q) f(q);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    for (int w = 0; w < nthreads; ++w)
        th.emplace_back([&] {
            for (;;) {
                int64_t q0 = next.fetch_add(64);
                if (q0 >= count) break;
                int64_t q1 = q0 + 64 < count ? q0 + 64 : count;
                for (int64_t q = q0; q < q1; ++q) f(q);
            }
        });
    for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

uint64_t ga_sim_derive_seed(uint64_t seed, uint64_t salt) { return derive(seed, salt); }

// make_reference (sim.py:60-65): codes 0..3 of "ACGT"
void ga_sim_reference(int64_t length, uint64_t seed, uint8_t* out) {
    MT rng;
    rng.seed_u64(derive(seed, 0x5EED));
    for (int64_t i = 0; i < length; ++i) out[i] = (uint8_t)std::floor(rng.random() * 4.0);
}

// simulate_read for one read: returns its length; writes codes if out != null
int64_t ga_sim_read(const uint8_t* ref, int64_t pos, int32_t length, double sub, double ins,
                    double dele, uint64_t seed, uint8_t* out) {
    return sim_one(ref, pos, length, sub, ins, dele, seed, out);
}

// simulate_read with its ground truth (sim.py:68-103, SimRecord): the read's
// codes and the edit script in reference order ('I', 'D', 'X', '='; up to
// 2 * length ops); returns the read length, *n_ops the script length
int64_t ga_sim_read_truth(const uint8_t* ref, int64_t pos, int32_t length, double sub, double ins,
                          double dele, uint64_t seed, uint8_t* out, char* ops, int64_t* n_ops) {
    return sim_one(ref, pos, length, sub, ins, dele, seed, out, ops, n_ops);
}

// CLI recipe positions (cli.py:141-144): read i has length read_lens[i]
void ga_sim_positions(int64_t ref_len, int64_t count, const int32_t* read_lens, uint64_t seed,
                      int64_t* pos_out) {
    MT rng;
    rng.seed_u64(derive(seed, 0xB0B));
    for (int64_t i = 0; i < count; ++i)
        pos_out[i] = (int64_t)rng.randbelow((uint64_t)(ref_len - read_lens[i] + 1));
}

// lengths of every read of the recipe (per-read seed derive_seed(seed, i+1))
void ga_sim_read_lengths(const uint8_t* ref, int64_t count, const int64_t* pos,
                         const int32_t* read_lens, double sub, double ins, double dele,
                         uint64_t seed, int nthreads, int32_t* out_len) {
    parallel_for(count, nthreads, [&](int64_t i) {
        out_len[i] = (int32_t)sim_one(ref, pos[i], read_lens[i], sub, ins, dele,
                                      derive(seed, (uint64_t)(i + 1)), nullptr);
    });
}

// fill pattern (read) and text (reference slice) codes at the given offsets
void ga_sim_fill_pairs(const uint8_t* ref, int64_t count, const int64_t* pos,
                       const int32_t* read_lens, double sub, double ins, double dele,
                       uint64_t seed, int nthreads, const int64_t* pat_off,
                       const int64_t* txt_off, uint8_t* codes) {
    parallel_for(count, nthreads, [&](int64_t i) {
        sim_one(ref, pos[i], read_lens[i], sub, ins, dele, derive(seed, (uint64_t)(i + 1)),
                codes + pat_off[i]);
        const uint8_t* src = ref + pos[i];
        uint8_t* dst = codes + txt_off[i];
        for (int32_t x = 0; x < read_lens[i]; ++x) dst[x] = src[x];
    });
}

}  // extern "C"
