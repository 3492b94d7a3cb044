/*
 * genasm.h -- C ABI of the B200-native improved-GenASM windowed aligner.
 *
 * The reference (`bitalign` 0.1.0, pure Python) has no FFI; its drop-in
 * boundary for the hot path is the Python API
 *     align(pattern, text, cfg)          pkg/src/bitalign/window.py:85-129
 *     align_batch(pairs, cfg, parallel)  pkg/src/bitalign/window.py:152-163
 *     WindowConfig                       pkg/src/bitalign/window.py:44-70
 *     AlignmentResult / BatchOutcome     pkg/src/bitalign/window.py:73-82, 132-141
 * The entry points below are what a binding of that API binds: one batched
 * call with plain pointers and sizes (no torch types), per-pair failures
 * returned as data (BatchOutcome.error), library errors as a return code +
 * ga_last_error().  The Python package paper_2203_15561_b200 binds this via
 * ctypes; INTEGRATION.md shows the stub a bitalign maintainer would add.
 *
 * Symbol codes (pkg/src/bitalign/distance.py:31, 70-79):
 *     0=A 1=C 2=G 3=T, 4=any other code unit (never matches, not even itself,
 *     lowercase included -- align() does not uppercase).
 */
#ifndef GENASM_H
#define GENASM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GA_MAX_WINDOW 128   /* kernel-supported window (configs need <= 128) */

/* Per-pair status (BatchOutcome.ok / .error; pkg/src/bitalign/window.py:144-149). */
enum {
    GA_OK = 0,
    GA_WINDOW_FAILED = 1,   /* "WindowFailed: window {i} found no alignment within k={k}" */
    GA_EMPTY_PATTERN = 2,   /* "EmptyPattern: pattern must not be empty" */
    GA_STUCK = 3,           /* StuckTraceback / PrunedAccess tripwire (never on valid tables) */
};

/* Driver parameters: WindowConfig (pkg/src/bitalign/window.py:44-70).
 * k must already be resolved (k=None -> window).  priority is a
 * permutation of "MSID" (pkg/src/bitalign/backtrace.py:64-67). */
typedef struct {
    int32_t window;
    int32_t overlap;
    int32_t k;
    char    priority[4];
    int32_t mode;      /* GA_MODE_IMPROVED (0) or GA_MODE_BASELINE (1): WindowConfig.mode */
} ga_config;

enum { GA_MODE_IMPROVED = 0, GA_MODE_BASELINE = 1 };

/* ga_batch_in.packed2 */
enum { GA_PACK_NONE = 0, GA_PACK_CALLER = 1, GA_PACK_HOST = 2 };

/* A batch of (pattern, text) pairs: the `pairs` list of align_batch.
 * All sequences live in one code array; offsets index into it. */
typedef struct {
    int64_t        n_pairs;
    const uint8_t* codes;      /* symbol codes 0..4 (one byte per symbol), or 2-bit
                                  packed ACGT when packed2 == GA_PACK_CALLER */
    int64_t        codes_len;  /* symbols in `codes`; must cover every offset + length
                                  (the device call converts exactly this range) */
    const int64_t* pat_off;    /* offsets and lengths are in symbols */
    const int32_t* pat_len;
    const int64_t* txt_off;
    const int32_t* txt_len;
    const int32_t* order;      /* optional processing order (a permutation of
                                  0..n_pairs-1, longest first for load balance);
                                  NULL: ga_align_batch computes it on the host,
                                  ga_align_batch_device uses input order.
                                  ga_align_batch checks it is a permutation (-3
                                  otherwise) and uses it only when the batch runs
                                  as one chunk: a chunked batch orders each chunk
                                  longest-first itself */
    /* ga_align_batch only, the input transfer format:
     * 0 (GA_PACK_NONE): `codes` are 1-byte codes, copied as they are;
     * 1 (GA_PACK_CALLER): 2-bit input, four symbols per byte (symbol x in
     *   bits 2(x%4)..2(x%4)+1 of byte x/4, 0..3 = ACGT); the positions of
     *   symbols outside ACGT (code 4) are listed in `exceptions` (ascending);
     * 2 (GA_PACK_HOST): `codes` are 1-byte codes; the call packs each
     *   pipeline chunk to 2 bits on the host (ga_pack2, into pinned staging)
     *   while the previous chunk's copy is in flight, and copies that --
     *   a quarter of the PCIe bytes.  n_exceptions/exceptions are ignored.
     * Other values return -3. */
    int32_t        packed2;
    int64_t        n_exceptions;
    const int64_t* exceptions;
} ga_batch_in;

/* One AlignmentResult (pkg/src/bitalign/window.py:73-82) or its failure.
 * 64 bytes, one D2H copy per batch. */
typedef struct {
    int32_t status;           /* GA_OK / GA_WINDOW_FAILED / GA_EMPTY_PATTERN / GA_STUCK */
    int32_t fail_window;      /* WindowFailed.window_index, else -1 */
    int64_t cost;             /* AlignmentResult.cost */
    int64_t text_consumed;    /* AlignmentResult.text_consumed */
    int64_t rows_computed;    /* AlignmentResult.rows_computed */
    int64_t ops_len;          /* len(AlignmentResult.cigar) */
    int64_t entry_reads;      /* AccessCounters.entry_reads   (dptable.py:85-105) */
    int64_t entry_writes;     /* AccessCounters.entry_writes */
    int64_t words_allocated;  /* AccessCounters.words_allocated */
} ga_pair_result;

/* Caller-allocated outputs.  ops_off/win_off are caller-computed prefix
 * sums: capacity pat_len+txt_len ops per pair and ga_num_windows() window
 * distances per pair. */
typedef struct {
    ga_pair_result* results;          /* n_pairs */
    const int64_t*  ops_off;          /* n_pairs, in ops */
    uint8_t*        ops;              /* ASCII '=','X','I','D' in walk (= forward) order,
                                         or 2-bit op codes when ops2 != 0; the whole
                                         capacity is written (bytes past a pair's
                                         ops_len are unspecified) */
    int64_t         ops_capacity;     /* ops that fit in `ops` */
    const int64_t*  win_off;          /* n_pairs */
    uint8_t*        window_distances; /* AlignmentResult.window_distances, d_min per window;
                                         0 for the windows a failed pair did not complete */
    int64_t         win_capacity;     /* entries in `window_distances` */
    /* ga_align_batch only: 2-bit ops (0 '=', 1 'X', 2 'I', 3 'D'), four per
     * byte like packed input; every ops_off must then be a multiple of 4. */
    int32_t         ops2;
} ga_batch_out;

typedef struct ga_ctx ga_ctx;

/* Library version string. */
const char* ga_version(void);

/* Number of windows align() walks for a pattern of length `pattern_len`
 * (1 + ceil(max(0, |P|-W)/(W-O)); 0 for an empty pattern). */
int64_t ga_num_windows(int64_t pattern_len, int32_t window, int32_t overlap);

/* Validate a config exactly as WindowConfig.__post_init__ plus the kernel's
 * window limit.  Returns 0 or writes a message into msg (may be NULL). */
int ga_check_config(const ga_config* cfg, char* msg, int msg_len);

/* Encode code units to symbol codes: 'A','C','G','T' -> 0..3, anything
 * else -> 4 (pkg/src/bitalign/distance.py:70-79: only the exact
 * uppercase alphabet has masks). */
void ga_encode_ascii(const char* seq, int64_t n, uint8_t* out);

/* The same on `threads` host threads (0: all): the drop-in Python
 * align_batch encodes its joined pair strings with it. */
void ga_encode_ascii_mt(const char* seq, int64_t n, uint8_t* out, int32_t threads);

/* ga_encode_ascii_mt over n_seqs separate ASCII buffers (ptrs[s], lens[s]),
 * written back to back into out (sum of lens bytes): the drop-in Python API
 * encodes the caller's str objects in place, with no joined copy. */
void ga_encode_ascii_gather(const uint64_t* ptrs, const int64_t* lens, int64_t n_seqs,
                            uint8_t* out, int32_t threads);

/* Create a context bound to one CUDA device (one context per device; a
 * context is not re-entrant).  Returns 0 or a CUDA error code. */
int ga_create(int device, ga_ctx** out);
void ga_destroy(ga_ctx* ctx);
const char* ga_last_error(const ga_ctx* ctx);

/* align_batch (pkg/src/bitalign/window.py:152-163) over HOST buffers:
 * host->device copies, the fused DC+TB kernel, device->host copies, pipelined
 * over chunks of consecutive pairs (copy-in / kernels / copy-out on separate
 * streams; GA_CHUNKS overrides the chunk count); returns when the results are
 * in `out`.  Results are in input order and independent of batch composition.
 * Pinned host buffers (ga_host_alloc) make the copies asynchronous. */
int ga_align_batch(ga_ctx* ctx, const ga_batch_in* in, const ga_config* cfg,
                   ga_batch_out* out);

/* Levenshtein distances of n pairs on the device -- the ground truth of the
 * `bench` accuracy columns: oracle.global_distance (semiglobal = 0) or
 * oracle.semiglobal_distance (semiglobal = 1; free text prefix),
 * pkg/src/bitalign/oracle.py:59-74.  in->codes holds symbol ids, one byte
 * per character (equal ids match, whatever the value -- unlike the
 * aligner's codes, where 4 never matches; see ga_pairs.syms in
 * genasm_io.h); packed2 is not supported.  dist[q] = the distance, or -1
 * for an empty pattern with semiglobal = 1 (the reference raises).
 * Synchronous. */
int ga_edit_distance(ga_ctx* ctx, const ga_batch_in* in, int32_t semiglobal, int64_t* dist);

/* Same call over DEVICE-resident buffers (every pointer in `in` and `out`
 * is a device pointer on the context's device).  Asynchronous on
 * `stream` (a cudaStream_t; NULL = the context's own stream).  1-byte codes
 * in, ASCII ops out: packed2 / ops2 return -3. */
int ga_align_batch_device(ga_ctx* ctx, const ga_batch_in* in, const ga_config* cfg,
                          ga_batch_out* out, void* stream);

/* Kernel launches issued by the last ga_align_batch* call (bench evidence). */
int64_t ga_last_launch_count(const ga_ctx* ctx);

/* Longest-first processing order (LPT) by pattern length: the host-side
 * length bucketing that balances mixed read lengths. */
void ga_lpt_order(int64_t n_pairs, const int32_t* pat_len, int32_t* order_out);

/* Host-side format helpers (multithreaded): 2-bit packing of symbol codes
 * into ceil(n/4) bytes; returns the number of code-4 symbols and lists the
 * first max_exceptions of their positions (ascending) in `exceptions` (may
 * be NULL to only count).  And 2-bit ops -> ASCII. */
int64_t ga_pack2(const uint8_t* codes, int64_t n, uint8_t* packed, int64_t* exceptions,
                 int64_t max_exceptions);
void ga_unpack_ops(const uint8_t* ops2, int64_t first_op, int64_t n_ops, char* out);

/* Pinned host memory for zero-staging host<->device copies (bench e2e). */
void* ga_host_alloc(int64_t bytes);
void ga_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* GENASM_H */
