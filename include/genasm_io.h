/*
 * genasm_io.h -- the file-format side of the `bitalign align` front-end, in
 * native code: pair-list TSV parsing straight into the ga_batch_in layout,
 * and the TSV result rows.  Exported by the same _genasm.so.
 *
 *   ga_parse_pairs_tsv   replaces io.read_pairs   pkg/src/bitalign/io.py:98-113
 *                        (plus the symbol coding of build_masks,
 *                        pkg/src/bitalign/distance.py:70-79)
 *   ga_format_align_rows replaces the row loop of cli._cmd_align
 *                        pkg/src/bitalign/cli.py:97-119 with io.format_cigar /
 *                        io.format_classic_cigar, io.py:142-175
 *
 * Host-only, multithreaded; no CUDA calls.
 */
#ifndef GENASM_IO_H
#define GENASM_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GA_IO_OK = 0,
    GA_IO_PARSE = 1,     /* PairParseError: err = "line N: <message>" (io.py:26-29) */
    GA_IO_NONASCII = 2,  /* a byte >= 0x80: decoding and str.upper() are Unicode-aware in the
                            reference; the caller parses such files with Python semantics */
    GA_IO_NOMEM = 3
};

/* A parsed pair list: the arrays ga_batch_in takes (codes 0..3 = ACGT after
 * ASCII upper-casing, 4 = any other code unit; pattern then text per pair,
 * concatenated) and the pair ids.  Owned by the library. */
typedef struct {
    int64_t        n_pairs;
    const uint8_t* codes;
    int64_t        codes_len;
    const int64_t* pat_off;
    const int32_t* pat_len;
    const int64_t* txt_off;
    const int32_t* txt_len;
    const char*    ids;     /* id bytes, concatenated */
    const int64_t* id_off;  /* n_pairs + 1 prefix sums into ids */
    const uint8_t* syms;    /* GA_PARSE_SYMBOLS: one symbol id per character, same layout as
                               codes; ids are a bijection of the upper-cased bytes (ACGT ->
                               0..3, bytes 0..3 -> 'A','C','G','T', others unchanged), so equal
                               ids <=> equal characters; NULL otherwise */
    void*          impl;    /* library-private */
} ga_pairs;

enum { GA_PARSE_SYMBOLS = 1 };

/* Parse `id<TAB>pattern<TAB>text` rows from a buffer holding a whole file.
 * Universal newlines (\n, \r\n, \r); blank lines and lines whose first
 * non-whitespace character is '#' are skipped but counted for line numbers;
 * a row with other than 3 columns or an empty pattern is a GA_IO_PARSE error
 * reporting the first such line.  nthreads <= 0: all hardware threads. */
int ga_parse_pairs_tsv(const char* data, int64_t len, int nthreads, int32_t flags,
                       ga_pairs** out, char* err, int64_t err_cap);
void ga_pairs_free(ga_pairs* pairs);

/* Flags of ga_format_align_rows */
enum { GA_ROWS_COLLAPSE_M = 1, GA_ROWS_STATS = 2 };

/* The stdout of `bitalign align` for n pairs (cli.py:104-118): per pair
 * `id\tcost\ttext_consumed\tcigar[\trows\treads\twrites\twords]\n`, or
 * `id\tERROR <error>\n` for a failed slot (window.py:144-149).  Ops as in
 * ga_batch_out: ASCII, or 2-bit when ops2 != 0.  Writes into buf and returns
 * the byte count, -1 if cap is too small (n * 200 + the id bytes + twice the
 * ops always suffice), -2 if a result carries status GA_STUCK (the reference
 * raises instead of writing a row). */
int64_t ga_format_align_rows(int64_t n, const char* ids, const int64_t* id_off, const void* results,
                             const uint8_t* ops, const int64_t* ops_off, int32_t ops2, int32_t k,
                             int32_t flags, int nthreads, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* GENASM_IO_H */
