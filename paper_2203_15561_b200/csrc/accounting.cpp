// accounting.cpp -- algorithmic work of a finished batch, for the roofline.
//
// From the outputs alone (cigar + window_distances) it
// rebuilds every window's geometry: window w of a pair covers the ops up to
// and including its (W-O)-th pattern-consuming op (traceback stops right
// after consuming its budget, pkg/src/bitalign/backtrace.py:117-121), so the
// text cursor t_w is the text consumed before it, n_w = min(W, |T| - t_w) and
// m_w = min(W, |P| - w(W-O)).  Sums:
//   entries  = sum (d_min+1) * n_w                 DC entries on levels <= d_min
//   alu_ops  = 5 * sum (d_min+1) * n_w * ceil(m_w/32)   int32 ops of the recurrence
//   cells    = sum m_w * n_w                       DP cells (GCUPS)
#include <stdint.h>

#include <atomic>
#include <thread>
#include <vector>

#include "../../include/genasm_bench.h"

extern "C" {

void ga_work_stats(const ga_batch_in* in, const ga_config* cfg, const ga_batch_out* out,
                   int nthreads, ga_work* total) {
    const int W = cfg->window, O = cfg->overlap;
    const int64_t n = in->n_pairs;
    if (nthreads < 1) nthreads = 1;
    std::vector<ga_work> part((size_t)nthreads, ga_work{0, 0, 0, 0, 0, 0});
    std::atomic<int64_t> next{0};
    auto work = [&](int tid) {
        ga_work acc{0, 0, 0, 0, 0, 0};
        for (;;) {
            int64_t q0 = next.fetch_add(256);
            if (q0 >= n) break;
            int64_t q1 = q0 + 256 < n ? q0 + 256 : n;
            for (int64_t q = q0; q < q1; ++q) {
                const ga_pair_result& r = out->results[q];
                if (r.status != GA_OK) continue;
                const int64_t Lp = in->pat_len[q], Lt = in->txt_len[q];
                const int64_t o0 = out->ops_off[q];
                // op x of the pair: ASCII, or 2-bit codes (0 '=', 1 'X', 2 'I', 3 'D')
                auto op_at = [&](int64_t x) -> uint8_t {
                    if (!out->ops2) return out->ops[o0 + x];
                    const int64_t y = o0 + x;
                    return "=XID"[(out->ops[y >> 2] >> (2 * (y & 3))) & 3];
                };
                const uint8_t* dist = out->window_distances + out->win_off[q];
                const int64_t nwin = ga_num_windows(Lp, W, O);
                int64_t pos = 0, t = 0;
                for (int64_t w = 0; w < nwin; ++w) {
                    const int64_t p = w * (int64_t)(W - O);
                    const int64_t m = Lp - p < W ? Lp - p : W;
                    const int64_t nn = Lt - t < W ? (Lt - t > 0 ? Lt - t : 0) : W;
                    const int64_t budget = (Lp - p <= W) ? m : W - O;
                    const int64_t lv = (int64_t)dist[w] + 1;
                    acc.windows++;
                    acc.entries += lv * nn;
                    acc.alu_ops += 5 * lv * nn * ((m + 31) / 32);
                    acc.cells += m * nn;
                    // walk this window's ops
                    int64_t consumed = 0;
                    while (pos < r.ops_len && consumed < budget) {
                        const uint8_t op = op_at(pos++);
                        if (op != 'D') consumed++;
                        if (op != 'I') t++;
                        acc.tb_steps++;
                    }
                }
                acc.pattern_bases += Lp;
            }
        }
        part[(size_t)tid] = acc;
    };
    std::vector<std::thread> th;
    for (int i = 0; i < nthreads; ++i) th.emplace_back(work, i);
    for (auto& x : th) x.join();
    ga_work s{0, 0, 0, 0, 0, 0};
    for (auto& p : part) {
        s.windows += p.windows;
        s.entries += p.entries;
        s.alu_ops += p.alu_ops;
        s.cells += p.cells;
        s.pattern_bases += p.pattern_bases;
        s.tb_steps += p.tb_steps;
    }
    *total = s;
}

}  // extern "C"
