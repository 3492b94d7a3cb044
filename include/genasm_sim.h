/*
 * genasm_sim.h -- workload generator exported by the same library: a
 * bit-exact port of the reference simulator so bench/parity inputs are the
 * pairs `bitalign simulate --emit-pairs` produces.
 *   ga_sim_derive_seed   pkg/src/bitalign/sim.py:53-57
 *   ga_sim_reference     pkg/src/bitalign/sim.py:60-65
 *   ga_sim_read          pkg/src/bitalign/sim.py:68-103
 *   ga_sim_read_truth    the same with SimRecord's edit script (truth_cigar)
 *   ga_sim_positions     pkg/src/bitalign/cli.py:141-144
 *   ga_sim_read_lengths, ga_sim_fill_pairs   pkg/src/bitalign/cli.py:145-169
 * Sequences are symbol codes 0..3 (ACGT), as in genasm.h.
 */
#ifndef GENASM_SIM_H
#define GENASM_SIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t ga_sim_derive_seed(uint64_t seed, uint64_t salt);
void ga_sim_reference(int64_t length, uint64_t seed, uint8_t* out);
int64_t ga_sim_read(const uint8_t* ref, int64_t pos, int32_t length, double sub, double ins,
                    double dele, uint64_t seed, uint8_t* out);
int64_t ga_sim_read_truth(const uint8_t* ref, int64_t pos, int32_t length, double sub, double ins,
                          double dele, uint64_t seed, uint8_t* out, char* ops, int64_t* n_ops);
void ga_sim_positions(int64_t ref_len, int64_t count, const int32_t* read_lens, uint64_t seed,
                      int64_t* pos_out);
void ga_sim_read_lengths(const uint8_t* ref, int64_t count, const int64_t* pos,
                         const int32_t* read_lens, double sub, double ins, double dele,
                         uint64_t seed, int nthreads, int32_t* out_len);
void ga_sim_fill_pairs(const uint8_t* ref, int64_t count, const int64_t* pos,
                       const int32_t* read_lens, double sub, double ins, double dele,
                       uint64_t seed, int nthreads, const int64_t* pat_off,
                       const int64_t* txt_off, uint8_t* codes);

#ifdef __cplusplus
}
#endif

#endif /* GENASM_SIM_H */
