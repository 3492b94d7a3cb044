/*
 * genasm_bench.h -- measurement helpers exported by the same library (used
 * by bench.py; not part of the alignment API).
 */
#ifndef GENASM_BENCH_H
#define GENASM_BENCH_H

#include <stdint.h>

#include "genasm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Algorithmic work of a finished batch, rebuilt from its outputs
 * (SURVEY 8(d), App. A.4): windows, DC entries sum (d_min+1)*n_w, int32 ALU
 * ops 5*sum (d_min+1)*n_w*ceil(m_w/32), DP cells sum m_w*n_w, pattern bases,
 * traceback steps. */
typedef struct {
    int64_t windows, entries, alu_ops, cells, pattern_bases, tb_steps;
} ga_work;

void ga_work_stats(const ga_batch_in* in, const ga_config* cfg, const ga_batch_out* out,
                   int nthreads, ga_work* total);

/* Measured int32 logic/shift issue peak of `device` in ops/s (best of reps). */
double ga_bench_alu_peak(int device, int reps);

#ifdef __cplusplus
}
#endif

#endif /* GENASM_BENCH_H */
