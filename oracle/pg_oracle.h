/*
 * pg_oracle.h -- plain-C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this (as the checker); the product never links it.
 *
 * Parity pinning: every function here is checked against the compiled reference
 * library (oracle/_ref/libpgref.so, tests/test_oracle.py) and against the reference
 * tests' known answers and committed golden fixtures (tests/golden/).
 *
 * Semantics follow the reference in parity mode (block size 1): the naive
 * dedispersion definition, not the defective multi-trial block path.
 */
#ifndef PG_ORACLE_H
#define PG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/pulsegrid_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int64_t pgo_delay_samples(double dm, const pgb_header* h, uint32_t channel);
double pgo_adaptive_dm_step(double tol, const pgb_header* h);
int pgo_generate_dm_trials(double dm_lo, double dm_hi, const pgb_header* h, int spacing,
                           double value, double* dms, int64_t* delays, size_t cap,
                           size_t* ntrials);

/* naive shift-and-add of one trial over a time-major float chunk */
void pgo_dedisperse(const float* data, uint64_t length, uint32_t nchans, const int64_t* delays,
                    float* out);
void pgo_remove_baseline(const float* x, uint64_t n, uint64_t window, float* out);
/* returns 0, or PGB_ERR_DEGENERATE; rms via *rms */
int pgo_normalize_to_sums(const float* x, uint64_t n, double* sums, double* rms);

int pgo_run_dm_loop_f32(const float* data, const pgb_chunk_spec* spec, uint32_t nchans,
                        const double* dms, const int64_t* delays, uint32_t ntrials,
                        const pgb_engine_config* cfg, pgb_candidate** cands, size_t* ncands,
                        uint64_t** skipped, size_t* nskipped);
int pgo_run_dm_loop_u8(const uint8_t* data, const pgb_chunk_spec* spec, uint32_t nchans,
                       const double* dms, const int64_t* delays, uint32_t ntrials,
                       const pgb_engine_config* cfg, pgb_candidate** cands, size_t* ncands,
                       uint64_t** skipped, size_t* nskipped);

void pgo_sort_candidates(pgb_candidate* c, size_t n);
int pgo_link_grid(const pgb_candidate* cands, size_t n, const pgb_link_radii* radii,
                  pgb_cluster** clusters, size_t* nclusters, uint64_t** members);
/* .cand text (src/cluster_io.cpp:11-34); returns bytes written (excl. NUL) */
size_t pgo_format_candidates(const pgb_cluster* clusters, size_t n, char* buf, size_t cap);

int pgo_plan_chunks(uint64_t nsamples, uint64_t chunk_len, uint64_t overlap, pgb_chunk_spec* out,
                    size_t cap, size_t* n);
void pgo_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
