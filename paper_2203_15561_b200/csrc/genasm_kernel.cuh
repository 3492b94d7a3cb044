// genasm_kernel.cuh -- launch interface of the fused windowed GenASM-DC +
// GenASM-TB kernels for sm_100a.
//
//   genasm_thread.cu (default, W <= 64): one pair per lane, DC in 32-bit
//     diagonal bands (genasm_thread.cuh), windows with d_min > 15 computed by
//     the whole warp as a levels-as-lanes wavefront.  DESIGN.md section 2.
//
//   genasm_lockstep.cu (W > 64, or GA_KERNEL=lockstep): every group of G lanes
//     owns one pair; the groups of a warp advance in PASS ROUNDS: each round,
//     every group runs one DC pass of its current window in lock-step (a
//     wavefront of G lanes x 16/G levels, R[d-1][j] passed by SHFL.UP), groups
//     whose window solved trace back together (G diagonal steps speculated per
//     ballot), set up their next window and rejoin.  A traceback state
//     (d, j, i) on any path from (d_min, n, m-1) satisfies
//     |(m-1-i) - (n-j)| <= d_min - d, so when d_min <= 15 a 32-bit band around
//     the diagonal holds every bit the traceback reads: band words per warp in
//     global memory, full-width rows in per-group slabs above level 15.
//
// Counters follow the reference's stored predicate (dptable.py:62-82) in
// closed form; entry reads are counted per taken step.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace genasm {

struct KernelParams {
    const uint8_t* codes;
    int64_t codes_len;         // symbols in codes
    // lane-per-pair kernel: the codes as three bit-planes (bit 0, bit 1, code 4),
    // plane_words 64-bit words each, built per launch by a streaming kernel
    const uint64_t* planes;
    int64_t plane_words;
    const int64_t* pat_off;
    const int32_t* pat_len;
    const int64_t* txt_off;
    const int32_t* txt_len;
    const int32_t* order;      // may be null (identity)
    int64_t n_pairs;
    int32_t W, O, k;
    uint32_t prio;             // 4 x 2-bit edge ids, first choice in bits 0-1 (0=M 1=S 2=I 3=D)
    uint64_t prio_lut;         // active-edge mask (M|S<<1|I<<2|D<<3) -> chosen edge, 4 bits each
    void* results;             // ga_pair_result[n_pairs]
    const int64_t* ops_off;
    uint8_t* ops;
    int64_t ops_capacity;
    const int64_t* win_off;
    uint8_t* dists;
    uint32_t* overflow;        // per-group global full-mode table slabs
    int64_t overflow_words_per_group;
    uint32_t* band;            // per-warp global band tables
    unsigned long long* queue; // atomic pair counter
    int32_t overlapped;        // 1: other launches share the GPU (pipeline chunks): keep no
                               // idle warps resident (lane-per-pair kernel)
};

struct PairResult {  // == ga_pair_result
    int32_t status, fail_window;
    int64_t cost, text_consumed, rows_computed, ops_len, entry_reads, entry_writes, words_allocated;
};

struct LaunchShape {
    int grid, block, smem_bytes, group, blocks_per_sm;
    int64_t overflow_words_per_group;
    int launches;  // kernels issued
};

// the unimproved engine (genasm_baseline.cu, mode="baseline"): all k+1 levels,
// dense 4-edge tables, one warp per pair
cudaError_t launch_genasm_baseline(KernelParams P, int num_sms, cudaStream_t stream,
                                   uint64_t** scratch, size_t* cap, LaunchShape* shape);

// Levenshtein distances for the accuracy columns (genasm_dp.cu)
cudaError_t launch_edit_distance(const uint8_t* syms, const int64_t* pat_off, const int32_t* pat_len,
                                 const int64_t* txt_off, const int32_t* txt_len, const int32_t* order,
                                 int64_t n_pairs, int max_words, int semiglobal, int64_t* dist,
                                 int num_sms, cudaStream_t stream, uint64_t** slab, size_t* cap,
                                 unsigned long long* queue);

// the fused kernel (genasm_lockstep.cu); group in {4, 8, 16} lanes per pair
cudaError_t launch_genasm_lockstep(const KernelParams& P, int group, int block_threads,
                                   int num_sms, cudaStream_t stream, uint32_t** overflow,
                                   size_t* cap, LaunchShape* shape);

// the lane-per-pair kernel (genasm_thread.cu), W <= 64; launches the
// bit-plane conversion of the codes first
cudaError_t launch_genasm_thread(const KernelParams& P, int num_sms, cudaStream_t stream,
                                 uint32_t** scratch, size_t* cap, LaunchShape* shape);

}  // namespace genasm
