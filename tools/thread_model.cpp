// thread_model.cpp -- dev tool: the lane-per-pair window code of
// csrc/genasm_thread.cuh run on the host, one pair at a time, so the band /
// full-tier math can be checked against the oracle without a GPU.
//   g++ -O2 -std=c++17 -shared -fPIC -o tools/_thread_model.so tools/thread_model.cpp
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "../include/genasm.h"
#include "../paper_2203_15561_b200/csrc/genasm_thread.cuh"

using namespace genasm::thr;

struct HostBand {
    using Word = uint32_t;
    static constexpr int kHalf = 16;
    std::vector<uint32_t> w;  // [column][8 paired words]
    void reset(int n) { w.assign((size_t)(n + 1) * 8, 0xdeadbeefu); }
    void put(int j, const uint32_t* pw) { memcpy(&w[(size_t)j * 8], pw, 32); }
    uint32_t get(int e, int c) const { return w[(size_t)c * 8 + packed_word(e)]; }
    uint32_t bit(uint32_t x, int e, int b) const { return packed_bit(x, e, b); }
};

struct HostWide {
    using Word = uint64_t;
    static constexpr int kHalf = 32;
    std::vector<uint32_t> w;  // [column][32 paired words]
    void reset(int n) { w.assign((size_t)(n + 1) * 32, 0xdeadbeefu); }
    void put4(int j, int q, const uint32_t* pw) { memcpy(&w[(size_t)j * 32 + 4 * q], pw, 16); }
    uint64_t get(int e, int c) const {
        const size_t k = (size_t)c * 32 + 2 * wide_pair(e);
        return (uint64_t)w[k + 1] << 32 | w[k];
    }
    uint32_t bit(uint64_t x, int e, int b) const { return wide_bit(x, e, b); }
};

struct HostFull {
    std::vector<uint64_t> w;  // [column][level]
    int LV = 0;
    void reset(int levels, int W) {
        LV = levels;
        w.assign((size_t)LV * (W + 1), 0x5555aaaa5555aaaaull);
    }
    void put4(int d0, int j, const uint32_t* lo, const uint32_t* hi) {
        for (int k = 0; k < 4; ++k) w[(size_t)j * LV + d0 + k] = (uint64_t)hi[k] << 32 | lo[k];
    }
    uint64_t get(int d, int j) const { return w[(size_t)j * LV + d]; }
};

extern "C" int model_align_batch(const ga_batch_in* in, const ga_config* cfg, ga_batch_out* out,
                                 int64_t* tier_counts) {
    const int W = cfg->window, O = cfg->overlap, K = cfg->k;
    if (W > 64) return -2;
    const uint64_t lut = make_prio_lut(cfg->priority);
    HostBand band;
    HostWide wide;
    HostFull full;
    const bool no_wide = getenv("MODEL_NO_WIDE") != nullptr;
    // the kernel's bit-plane form of the codes
    const int64_t pw = (in->codes_len + 63) / 64 + 1;
    std::vector<uint64_t> pl((size_t)pw * 3, 0);
    for (int64_t x = 0; x < in->codes_len; ++x) {
        const uint8_t c = in->codes[x];
        pl[x >> 6] |= (uint64_t)(c & 1) << (x & 63);
        pl[pw + (x >> 6)] |= (uint64_t)((c >> 1) & 1) << (x & 63);
        pl[2 * pw + (x >> 6)] |= (uint64_t)((c >> 2) & 1) << (x & 63);
    }
    for (int64_t q = 0; q < in->n_pairs; ++q) {
        ga_pair_result& r = out->results[q];
        memset(&r, 0, sizeof r);
        r.fail_window = -1;
        const int Lp = in->pat_len[q], Lt = in->txt_len[q];
        const uint8_t* P = in->codes + in->pat_off[q];
        const uint8_t* T = in->codes + in->txt_off[q];
        uint8_t* ops = out->ops + out->ops_off[q];
        uint8_t* dists = out->window_distances + out->win_off[q];
        if (Lp <= 0) {
            r.status = GA_EMPTY_PATTERN;
            continue;
        }
        int64_t p = 0, t = 0, nops = 0;
        int widx = 0;
        int status = GA_OK;
        while (p < Lp) {
            const int64_t rem = Lp - p;
            const bool fin = rem <= W;
            const int m = fin ? (int)rem : W;
            const int64_t tl = Lt - t;
            const int n = tl < W ? (int)(tl > 0 ? tl : 0) : W;
            const int budget = fin ? m : W - O;
            int d_min;
            TbOut o{};
            bool ok = true;
            if (n == 0) {
                if (m > K) {
                    status = GA_WINDOW_FAILED;
                    break;
                }
                d_min = m;
                Planes pp = load_planes_bits(pl.data(), pw, in->pat_off[q] + p, m), tp{0, 0, 0};
                ok = traceback([&](int, int, int) -> uint32_t { return 1u; }, pp, tp, m, n, d_min,
                               budget, lut, ops, nops, o);
                tier_counts[2]++;
            } else {
                Planes pp = load_planes_bits(pl.data(), pw, in->pat_off[q] + p, m),
                       tp = load_planes_bits(pl.data(), pw, in->txt_off[q] + t, n);
                band.reset(n);
                uint32_t okm = dc_band(pp, tp, m, n, band_jstore(n, budget), band);
                const int lim = K < 15 ? K : 15;
                okm &= (2u << lim) - 1u;
                if (okm) {
                    d_min = __builtin_ctz(okm);
                    ok = tb_band_t(band, pp, tp, m, n, d_min, budget, lut, ops, nops, o);
                    tier_counts[0]++;
                } else if (K <= 15) {
                    status = GA_WINDOW_FAILED;
                    break;
                } else {
                    uint32_t wm = 0;
                    if (!no_wide) {
                        wide.reset(n);
                        wm = dc_wide(pp, tp, m, n, wide_jstore(n, budget), wide);
                        wm &= K < 31 ? (2u << K) - 1u : ~0u;
                        if (wm & 0xffffu) return -10;  // the band tier is exact below 16
                    }
                    if (wm) {
                        d_min = __builtin_ctz(wm);
                        ok = tb_band_t(wide, pp, tp, m, n, d_min, budget, lut, ops, nops, o);
                        tier_counts[3]++;
                        goto booked;
                    }
                    if (!no_wide && K <= 31) {
                        status = GA_WINDOW_FAILED;
                        break;
                    }
                    full.reset((K + kPassLevels) / kPassLevels * kPassLevels, W);
                    d_min = dc_full(pp, tp, m, n, K, full);
                    if (d_min < 0) {
                        status = GA_WINDOW_FAILED;
                        break;
                    }
                    ok = traceback([&](int e, int c, int x) { return full_bit(full, e, c, x); },
                                   pp, tp, m, n, d_min, budget, lut, ops, nops, o);
                    tier_counts[1]++;
                }
            }
        booked:
            if (!ok) {
                status = GA_STUCK;
                break;
            }
            const int64_t wr = window_writes(n, budget, K, d_min);
            dists[widx] = (uint8_t)d_min;
            r.rows_computed += d_min + 1;
            r.cost += o.wcost;
            r.entry_reads += o.reads;
            r.entry_writes += wr;
            r.words_allocated += wr * ((m + 63) / 64);
            p += o.consumed;
            t += o.tcons;
            ++widx;
        }
        if (status != GA_OK) {
            memset(&r, 0, sizeof r);
            r.status = status;
            r.fail_window = widx;
            continue;
        }
        r.text_consumed = t;
        r.ops_len = nops;
    }
    return 0;
}
