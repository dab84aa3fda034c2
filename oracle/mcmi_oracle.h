/* oracle/mcmi_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, serial restatement of the reference preconditioner build
 * (mcspai::compute_preconditioner_serial, /root/reference/proj/src/mc_engine.cpp:153-238)
 * used as the parity checker for the CUDA path.  Besides the reference's own
 * RNG keying ("reference" mode: one Philox stream per row, draws numbered
 * across chains, rng.hpp:17-74 / mc_engine.cpp:168) it implements the keyed
 * mode u(row, chain, step) that the B200 kernel uses for chain parallelism.
 * Parity of this restatement is pinned against the reference library itself
 * (oracle/_ref) and the golden hashes in BASELINE.md — see tests/test_oracle.py.
 *
 * Never linked into, loaded by, or called from the product path.
 */
#ifndef MCMI_ORACLE_H
#define MCMI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same field layout as mcmi_config (include/mcmi.h). */
typedef struct orc_config {
    double epsilon;
    double delta;
    double alpha;
    int32_t mode;      /* 0 plain, 1 sign_aware */
    int32_t drop_mode; /* 0 value_range, 1 count_quantile */
    double drop_fraction;
    int64_t retain_k;
    int32_t has_chains_override;
    int32_t has_max_len_override;
    int64_t chains_override;
    int64_t max_len_override;
    uint64_t master_seed;
    int32_t rng_mode; /* 0 reference stream, 1 keyed (row, chain, step) */
    int32_t device;   /* ignored */
    int32_t flags;    /* ignored (the oracle always counts) */
    int32_t n_gpus;   /* ignored */
} orc_config;

typedef struct orc_result orc_result;

/* status: 0 ok, 1 invalid_argument, 2 split error, 5 out of memory */
int orc_build(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
              const orc_config* cfg, int64_t row_begin, int64_t row_end, orc_result** out,
              char* err, size_t errlen);
void orc_result_sizes(const orc_result* r, int64_t* n_rows, int64_t* nnz);
void orc_result_copy(const orc_result* r, int64_t* row_ptr, int64_t* col_idx, double* values,
                     int64_t* chains_used, int64_t* entries_before, int64_t* n_chains,
                     int64_t* max_len, int64_t* walk_steps, int64_t* walk_deg_sum,
                     double* a_norm);
void orc_result_free(orc_result* r);

/* Philox4x32-10 block (rng.hpp:44-67). */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif
