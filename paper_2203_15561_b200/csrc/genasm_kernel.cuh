// genasm_kernel.cuh -- fused windowed GenASM-DC + GenASM-TB for sm_100a.
//
// Work mapping.  A persistent grid; every warp holds 32/G pairs, one per GROUP
// of G consecutive lanes (G = 8 by default).  Groups pull pairs from an atomic
// queue (longest first) and walk the reference's sequential window chain
// (pkg/src/bitalign/window.py:95-120).  The groups of a warp advance in
// PASS ROUNDS: every round, every group runs one DC pass of its current
// window in lock-step (no divergence on the hot loop); groups whose window
// solved in that pass then trace back together, set up their next window (or
// pull the next pair) and rejoin at the next round.
//
//   DC pass (pkg/src/bitalign/distance.py:97-150): a wavefront of G lanes that
//     covers 16 levels; lane q owns LPL = 16/G consecutive levels and at step s
//     evaluates column j = s-q+1 of all of them, column-major inside the lane.
//     The first of its levels takes R[d-1][j] from lane q-1 by one warp
//     shuffle (lane 0: the carry row of the previous pass, full-width rows of
//     its last level).  Rows are NW x 32-bit registers (W <= 32 NW).  Early
//     termination (key idea 2): the window's DC ends with the first pass
//     holding a level whose column-n row has bit m-1 clear.  The table keeps
//     one status row per entry -- the AND of the four edges (key idea 1).
//
//   Table (key idea 3, extended to bits).  A traceback state (d, j, i) on any
//     path from (d_min, n, m-1) satisfies |(m-1-i) - (n-j)| <= d_min - d, so
//     every table read of entry (e, j) touches bits within d_min - e of the
//     diagonal c_j = m-1-n+j.  When d_min <= 15 a 32-bit band around c_j holds
//     every bit the traceback can ever read: band mode stores 32 bits per entry
//     for levels 0..15, in a per-warp global region laid out [pass][step][lane]
//     x LPL words so each wavefront step is one coalesced 16-byte store per
//     lane (the region stays L2-resident).  A window needing level 16+ restarts
//     in full mode (full-width rows in a per-group global slab).  W <= 32 rows
//     are 32 bits wide and need no band.
//
//   TB (pkg/src/bitalign/backtrace.py:70-167): greedy walk from
//     (j=n, d=d_min, i=m-1), edge bits recomputed from three table reads and
//     the symbol codes (backtrace.py:84-99), first active edge by a priority
//     LUT.  The G lanes speculate G consecutive diagonal ('=') steps at once;
//     a ballot finds the first non-match, so a run of matches costs one round
//     trip.  Ops are emitted in walk (= forward) order.
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
    const int64_t* win_off;
    uint8_t* dists;
    uint32_t* overflow;        // per-group global full-mode table slabs
    int64_t overflow_words_per_group;
    uint32_t* band;            // per-warp global band tables
    unsigned long long* queue; // atomic pair counter
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

// the fused kernel (genasm_lockstep.cu); group in {4, 8, 16} lanes per pair
cudaError_t launch_genasm_lockstep(const KernelParams& P, int group, int block_threads,
                                   int num_sms, cudaStream_t stream, uint32_t** overflow,
                                   size_t* cap, LaunchShape* shape);

// the lane-per-pair kernel (genasm_thread.cu), W <= 64; launches the
// bit-plane conversion of the codes first
cudaError_t launch_genasm_thread(const KernelParams& P, int num_sms, cudaStream_t stream,
                                 uint32_t** scratch, size_t* cap, LaunchShape* shape);

}  // namespace genasm
