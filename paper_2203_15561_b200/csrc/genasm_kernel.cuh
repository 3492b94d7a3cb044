// genasm_kernel.cuh -- fused windowed GenASM-DC + GenASM-TB for sm_100a.
//
// One pair per GROUP of G lanes (G = 8/16/32; 32/G pairs per warp).  A
// persistent grid pulls pairs from an atomic queue in longest-first order.
// Per pair the lanes walk the reference's sequential window chain
// (pkg/src/bitalign/window.py:95-120); per window:
//
//   DC (pkg/src/bitalign/distance.py:97-150): levels-as-lanes wavefront.
//     Pass p evaluates levels pG..pG+G-1, lane q owns level d = pG+q and at
//     step s computes column j = s-q+1, receiving R[d-1][j] from lane q-1
//     by one warp shuffle (lane 0 reads level pG-1 back from the table).
//     Rows are NW x 32-bit registers (W <= 32*NW).  Early termination (key
//     idea 2): the first pass containing a level whose column-n row has bit
//     m-1 clear ends the DC; d_min is the lowest such level.  The table
//     keeps exactly one status row per entry, the AND of the four edges
//     (key idea 1).
//   TB (pkg/src/bitalign/backtrace.py:70-167): greedy walk from
//     (j=n, d=d_min, i=m-1), edge bits recomputed from three table reads
//     (backtrace.py:84-99) and the symbol codes, first active edge in the
//     configured priority.  Ops are emitted in walk (= forward) order.
//
// Table placement: levels < S_LV live in shared memory, the rest in a
// per-group global overflow slab.  Counters follow the reference's stored
// predicate (dptable.py:62-82) in closed form.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace genasm {

struct KernelParams {
    const uint8_t* codes;
    const int64_t* pat_off;
    const int32_t* pat_len;
    const int64_t* txt_off;
    const int32_t* txt_len;
    const int32_t* order;      // may be null (identity)
    int64_t n_pairs;
    int32_t W, O, k;
    uint32_t prio;             // 4 x 2-bit edge ids, first choice in bits 0-1 (0=M 1=S 2=I 3=D)
    void* results;             // ga_pair_result[n_pairs]
    const int64_t* ops_off;
    uint8_t* ops;
    const int64_t* win_off;
    uint8_t* dists;
    uint32_t* overflow;        // per-group global table slabs
    int64_t overflow_words_per_group;
    int32_t s_lv;              // table levels resident in shared memory
    unsigned long long* queue; // atomic pair counter
};

struct PairResult {  // == ga_pair_result
    int32_t status, fail_window;
    int64_t cost, text_consumed, rows_computed, ops_len, entry_reads, entry_writes, words_allocated;
};

struct LaunchShape {
    int grid, block, smem_bytes, s_lv, group;
    int64_t overflow_words_per_group;
};

cudaError_t launch_genasm(const KernelParams& P, int group, int s_lv, int smem_budget, int num_sms,
                          cudaStream_t stream, uint32_t** overflow, size_t* cap,
                          LaunchShape* shape);

}  // namespace genasm
