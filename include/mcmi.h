/* include/mcmi.h — C-ABI of the B200 MCMCMI preconditioner builder.
 *
 * Drop-in boundary for the reference's preconditioner-build path:
 *
 *   mcspai::ApproxInverse mcspai::compute_preconditioner(const CsrMatrix& b,
 *                                                        const McConfig& cfg,
 *                                                        int n_threads = 0);
 *   (/root/reference/proj/include/mcspai/mc_engine.hpp:80-81,
 *    implementation src/mc_engine.cpp:153-233)
 *
 * The reference passes std::vector-backed CSR (int64 indices, f64 values,
 * csr.hpp:10-21) by const reference and returns the result by value.  A C ABI
 * cannot return an unknown-size value, so the host entry point returns an
 * opaque result handle: build -> query sizes -> copy out -> free
 * (mcmi_build / mcmi_result_sizes / mcmi_result_copy / mcmi_result_free).
 * Reference exceptions map to status codes (see MCMI_E*); the message text is
 * the reference's own (mc_engine.cpp:14, split.cpp:48,68,95, csr.cpp:129).
 * include/mcmi/mcspai_compat.hpp re-throws them as the same C++ types.
 *
 * The device-resident engine (mcmi_engine_*) is the same pipeline with inputs
 * and outputs in HBM, used for sharded multi-GPU builds and for timing.
 *
 * All entry points are reentrant; one engine must not be used by two host
 * threads at once.
 */
#ifndef MCMI_H
#define MCMI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCMI_ABI_VERSION 1

/* status codes */
#define MCMI_OK 0
#define MCMI_EINVAL 1  /* std::invalid_argument (drop fraction, alpha, ||A|| range, bad config) */
#define MCMI_ESPLIT 2  /* mcspai::SplitError (degenerate diagonal, dominance failure) */
#define MCMI_ERANGE 3  /* std::out_of_range (column index outside [0, n)) */
#define MCMI_ECUDA 4   /* CUDA runtime failure */
#define MCMI_ENOMEM 5  /* device or host allocation failure */
#define MCMI_ENODEV 6  /* no CUDA device / device ordinal invalid */
#define MCMI_EPARSE 7  /* mcspai::ParseError (matrix_market.hpp:12-14), message names the line */
#define MCMI_EIO 8     /* std::runtime_error from file I/O (cannot open / write failure) */
#define MCMI_ERECOVERY 9 /* mcspai::RecoveryError (recovery.hpp:9-11): "singular update at row i" */

/* AugmentationMode (split.hpp:9-12) */
#define MCMI_AUGMENT_PLAIN 0
#define MCMI_AUGMENT_SIGN_AWARE 1
/* DropMode (csr.hpp:61-64) */
#define MCMI_DROP_VALUE_RANGE 0
#define MCMI_DROP_COUNT_QUANTILE 1
/* RNG keying of the walks */
#define MCMI_RNG_REFERENCE 0 /* RngStream(seed, row), draws numbered across chains:
                                byte-identical to the reference (mc_engine.cpp:168) */
#define MCMI_RNG_KEYED 1     /* u(row, chain, step) = Philox({step>>1, chain, row}, seed) */

/* Mirror of mcspai::McConfig (mc_engine.hpp:15-26).  std::optional fields are
 * split into has_* flags; every int64 value is meaningful, as in the reference. */
typedef struct mcmi_config {
    double epsilon;       /* default 0.0625 */
    double delta;         /* default 0.0625 */
    double alpha;         /* default 5.0 */
    int32_t mode;         /* MCMI_AUGMENT_*, default sign_aware */
    int32_t drop_mode;    /* MCMI_DROP_*, default value_range */
    double drop_fraction; /* default 0.0 */
    int64_t retain_k;     /* 0 = unlimited */
    int32_t has_chains_override;
    int32_t has_max_len_override;
    int64_t chains_override;
    int64_t max_len_override;
    uint64_t master_seed;
    int32_t rng_mode; /* MCMI_RNG_*, default MCMI_RNG_REFERENCE */
    int32_t device;   /* CUDA device ordinal for mcmi_build */
    int32_t flags;    /* MCMI_FLAG_*, default 0 */
    int32_t n_gpus;   /* host builds (mcmi_build*): row blocks on devices device..device+n_gpus-1,
                         one host thread each; 0 = env MCMI_GPUS (default 1).  M does not
                         depend on it.  The device-resident engine ignores it. */
} mcmi_config;

/* flags */
#define MCMI_FLAG_DEG_STATS 1 /* also count sum of deg(s) over walk steps (mcmi_stats.walk_deg_sum);
                                 costs ~4% walk throughput (registers), so it is opt-in */
#define MCMI_FLAG_UNSCALED 2  /* rows of (I - A)^-1 as mcspai::estimate_row returns them
                                 (mc_engine.hpp:57-65): no scale_columns, no zero prune.  With
                                 retain_k = 0 and rows (r, r+1) this is estimate_row(split, r,
                                 budget, delta, RngStream(master_seed, r)). */

/* Fills cfg with the reference defaults (McConfig{}). */
void mcmi_config_default(mcmi_config* cfg);

/* Square CSR in the reference layout (csr.hpp:16-21): row_ptr[n+1],
 * col_idx[nnz], values[nnz], nnz = row_ptr[n].  Host pointers for mcmi_build,
 * device pointers for mcmi_engine_build. */
typedef struct mcmi_csr_view {
    int64_t n;
    const int64_t* row_ptr;
    const int64_t* col_idx;
    const double* values;
} mcmi_csr_view;

/* Per-build statistics (not in the reference; budget_echo is ChainBudget,
 * mc_engine.hpp:28-31). */
typedef struct mcmi_stats {
    int64_t n_chains;     /* ChainBudget::n_chains */
    int64_t max_len;      /* ChainBudget::max_len */
    double a_norm;        /* SplitSystem::a_norm */
    int64_t rows;         /* rows built (row_end - row_begin) */
    int64_t nnz;          /* entries of the built rows of M */
    int64_t walk_steps;   /* sampled transitions (one per s->t move) */
    int64_t walk_deg_sum; /* sum over steps of deg(s) (MCMI_FLAG_DEG_STATS, else -1):
                             algorithmic bytes = 20*steps + 8*deg_sum */
    int64_t hash_cap;     /* accumulator capacity of the first tier */
    int64_t rows_retried; /* rows re-run on a larger accumulator tier */
    double ms_tables;     /* device time: drop + split + transition tables */
    double ms_walk;       /* device time: walk + accumulate + finalize kernels */
    double ms_assemble;   /* device time: row-pointer scan + CSR compaction */
    double ms_total;      /* device time of the whole build (excl. host copies) */
    int64_t launches;     /* kernels launched by this build */
    double ms_walk_kernel; /* device time of the walk kernel launches alone */
} mcmi_stats;

/* ------------------------------------------------------------ host API */

typedef struct mcmi_result mcmi_result;

/* compute_preconditioner: host CSR in, host result out.  B may be pageable
 * (staged through pinned bounce buffers) or page-locked.  The result is
 * host-resident in library-owned page-locked arrays (pooled across builds),
 * filled by a streamed build: each row chunk's device->host copy overlaps the
 * next chunk's walks.  No output size is needed in advance. */
int mcmi_build(const mcmi_csr_view* b, const mcmi_config* cfg, mcmi_result** out, char* err,
               size_t errlen);
/* Same, restricted to rows [row_begin, row_end) of M (a row shard: the
 * result's row_ptr starts at 0, RowMeta covers only those rows).  The
 * transition tables always cover all n states. */
int mcmi_build_rows(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin,
                    int64_t row_end, mcmi_result** out, char* err, size_t errlen);
/* Streamed variant: builds rows [row_begin, row_end) straight into caller-owned
 * host arrays (pinned memory gives full PCIe bandwidth), overlapping the
 * device->host copy of each row chunk with the walks of the next.  row_ptr
 * [rows+1]; col_idx / values hold `capacity` entries; chains_used /
 * entries_before [rows] may be NULL.  *nnz receives the entry count; if it
 * exceeds capacity the call returns MCMI_ENOMEM (and *nnz says how much is
 * needed).  Same results as mcmi_build_rows. */
int mcmi_build_into(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin, int64_t row_end,
                    int64_t* row_ptr, int64_t* col_idx, double* values, int64_t capacity,
                    int64_t* chains_used, int64_t* entries_before, int64_t* nnz, mcmi_stats* stats,
                    char* err, size_t errlen);
/* ------------------------------------------- fine-grained pipeline stages */
/* The reference's public building blocks, on the same device
 * code as the build.  retain_top_k / scale_columns are fused into the walk's
 * per-row finalize (MCMI_FLAG_UNSCALED returns the rows before them). */

/* mcspai::derive_chain_budget (mc_engine.hpp:55, mc_engine.cpp:12-33), host
 * arithmetic (glibc log / ceil) as in the build.  MCMI_EINVAL: "||A|| must lie
 * in [0,1)". */
int mcmi_derive_chain_budget(const mcmi_config* cfg, double a_norm, int64_t* n_chains, int64_t* max_len, char* err,
                             size_t errlen);

/* mcspai::augment_and_split (split.hpp:34-35, split.cpp:46-100) with
 * transition_probabilities (split.cpp:102-119), computed on `device`; the
 * result is copied to host memory.  Errors: MCMI_EINVAL "alpha must be
 * positive"; MCMI_ESPLIT degenerate diagonal / dominance failure (the
 * reference's messages); MCMI_ERANGE for a column outside [0, n) (the
 * reference does not check). */
typedef struct mcmi_split_system mcmi_split_system;
int mcmi_augment_and_split(const mcmi_csr_view* b, double alpha, int32_t mode, int device, mcmi_split_system** out,
                           char* err, size_t errlen);
/* n, entries of b_hat and of A (P has A's pattern), ||A||inf */
int mcmi_split_sizes(const mcmi_split_system* s, int64_t* n, int64_t* nnz_b_hat, int64_t* nnz_a, double* a_norm);
/* Any pointer may be NULL.  b_hat: row_ptr[n+1], col_idx / values[nnz_b_hat];
 * b1_diag[n]; A: row_ptr[n+1], col_idx / values[nnz_a]; p_values[nnz_a];
 * s_diag[n] (SplitSystem, split.hpp:21-28). */
int mcmi_split_copy(const mcmi_split_system* s, int64_t* b_hat_row_ptr, int64_t* b_hat_col_idx, double* b_hat_values,
                    double* b1_diag, int64_t* a_row_ptr, int64_t* a_col_idx, double* a_values, double* p_values,
                    double* s_diag);
void mcmi_split_free(mcmi_split_system* s);

/* mcspai::estimate_row (mc_engine.hpp:63-65, mc_engine.cpp:80-122) on a
 * caller-built SplitSystem, for rows [row_begin, row_end) at once: a = split.a
 * (host CSR), p_values = split.p's values on A's pattern (nnz(A) doubles),
 * budget (n_chains >= 1, max_len), delta, and row r's stream RngStream(seed, r)
 * (rng_mode MCMI_RNG_REFERENCE) or the keyed stream.  Row r of the result is
 * exactly estimate_row's SparseRow: columns sorted, values unscaled, nothing
 * pruned or retained (b1_diag is not needed).  The tables are built from A and
 * P on `device` per call (O(nnz) there; estimate_row itself allocates O(n)
 * per call, mc_engine.cpp:120).  Result: as mcmi_build_rows (RowMeta
 * chains_used = chains_run). */
int mcmi_estimate_rows(const mcmi_csr_view* a, const double* p_values, int64_t row_begin, int64_t row_end,
                       int64_t n_chains, int64_t max_len, double delta, uint64_t seed, int32_t rng_mode, int device,
                       mcmi_result** out, char* err, size_t errlen);

/* mcspai::retain_top_k (mc_engine.hpp:70, mc_engine.cpp:124-145) on every row
 * of a host CSR at once (each row one SparseRow): row r keeps the k entries
 * ranked first by (column == diag_cols[r] first, |value| descending, column
 * ascending), in their original order; rows with <= k entries, and every row
 * when k <= 0, are unchanged.  diag_cols NULL means diag_cols[r] = r.
 * out_row_ptr[n+1]; out_col_idx / out_values hold nnz(rows) entries; *out_nnz
 * = entries kept.  (The build applies the same rule inside the walk kernel.) */
int mcmi_retain_top_k(const mcmi_csr_view* rows, int64_t k, const int64_t* diag_cols, int device,
                      int64_t* out_row_ptr, int64_t* out_col_idx, double* out_values, int64_t* out_nnz, char* err,
                      size_t errlen);
/* mcspai::scale_columns (mc_engine.hpp:74, mc_engine.cpp:147-149) on every
 * entry of a host CSR: out_values[i] = values[i] / b1_diag[col_idx[i]].
 * MCMI_ERANGE if a column is outside [0, b1_len) (the reference indexes
 * without a check). */
int mcmi_scale_columns(const mcmi_csr_view* rows, const double* b1_diag, int64_t b1_len, int device,
                       double* out_values, char* err, size_t errlen);

/* mcspai::transition_probabilities (split.hpp:39) of any CSR A on `device`:
 * p_ij = |a_ij| / sequential row sum; rows summing to 0 become empty.
 * p_row_ptr[n+1]; p_col_idx / p_values hold nnz(A) entries; *p_nnz = entries
 * written. */
int mcmi_transition_probabilities(const mcmi_csr_view* a, int device, int64_t* p_row_ptr, int64_t* p_col_idx,
                                  double* p_values, int64_t* p_nnz, char* err, size_t errlen);

/* mcspai::drop_small_entries (csr.hpp:76-77, csr.cpp:127-157) on `device`:
 * the build's drop filter as a matrix.  out_row_ptr[n+1]; out_col_idx /
 * out_values hold nnz(m) entries; *out_nnz = entries kept.  MCMI_EINVAL:
 * "drop fraction must lie in [0,1]". */
int mcmi_drop_small_entries(const mcmi_csr_view* m, double p, int32_t drop_mode, int device, int64_t* out_row_ptr,
                            int64_t* out_col_idx, double* out_values, int64_t* out_nnz, char* err, size_t errlen);

/* Row blocks of a sharded build: edges[0..parts] with block g =
 * rows [edges[g], edges[g+1]) of [row_begin, row_end), balanced on cost(r) =
 * 1 + nnz(r); edges[g] (0 < g < parts) is the first row whose cost prefix
 * reaches total*g/parts.  Used by host builds with n_gpus > 1 and by the
 * one-process-per-GPU driver (distributed.partition_rows).  Host only. */
int mcmi_partition_rows(const int64_t* row_ptr, int64_t row_begin, int64_t row_end, int parts, int64_t* edges);
/* The same build of rows [row_begin, row_end) started on a library thread, for
 * callers that size their own output while the walks run (the C++ drop-in,
 * include/mcmi/mcspai_compat.hpp): B's arrays must stay valid until
 * mcmi_job_finish.  mcmi_job_estimate blocks until the first row chunk (5% of
 * the rows) is built and returns an upper-biased extrapolation of nnz(M)
 * (x1.08 + 1024; exact when the build has a single chunk or is over), or -1
 * with the build's error status if it failed first; later calls return at once
 * with the latest estimate (refreshed after every chunk, never lowered).  mcmi_job_finish waits for the
 * build and returns its result (to be freed with mcmi_result_free), or the
 * build's error; it frees the job. */
typedef struct mcmi_job mcmi_job;
int mcmi_build_start(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin, int64_t row_end,
                     mcmi_job** job, char* err, size_t errlen);
int mcmi_job_estimate(mcmi_job* job, int64_t* nnz_estimate);
/* Hands the job the caller's entry arrays, of which entries [0, capacity) may
 * be written: from then on every row chunk is copied into them as soon as its
 * device->host copy completes, while later chunks still walk.  May be called
 * again with the same arrays and a larger capacity as the caller's storage
 * grows.  Entries beyond `capacity` are not delivered (mcmi_result_copy_range
 * copies them later). */
int mcmi_job_attach(mcmi_job* job, int64_t* col_idx, double* values, int64_t capacity);
/* *delivered (may be NULL) = the leading entries already in the attached
 * arrays; the rest is copied with mcmi_result_copy_range. */
int mcmi_job_finish(mcmi_job* job, mcmi_result** out, int64_t* delivered, char* err, size_t errlen);

int mcmi_result_sizes(const mcmi_result* r, int64_t* n, int64_t* nnz);
/* Any pointer may be NULL.  row_ptr[n+1], col_idx[nnz], values[nnz],
 * chains_used[n] / entries_before[n] = RowMeta (mc_engine.hpp:33-36),
 * n_chains / max_len = budget_echo.  A multi-threaded host copy. */
int mcmi_result_copy(const mcmi_result* r, int64_t* row_ptr, int64_t* col_idx, double* values,
                     int64_t* chains_used, int64_t* entries_before, int64_t* n_chains,
                     int64_t* max_len);
/* Entries [begin, end) of col_idx / values (either may be NULL) into
 * col_idx[begin..end) / values[begin..end): a multi-threaded host copy. */
int mcmi_result_copy_range(const mcmi_result* r, int64_t begin, int64_t end, int64_t* col_idx, double* values);
/* Borrowed pointers to the result's host arrays (valid until mcmi_result_free;
 * col_idx / values are NULL when nnz == 0): zero-copy access for bindings. */
int mcmi_result_view(const mcmi_result* r, const int64_t** row_ptr, const int64_t** col_idx, const double** values,
                     const int64_t** chains_used, const int64_t** entries_before);
int mcmi_result_stats(const mcmi_result* r, mcmi_stats* stats);
void mcmi_result_free(mcmi_result* r);

/* ---------------------------------------------------- device-resident API */

typedef struct mcmi_engine mcmi_engine;

/* Device CSR shard produced by mcmi_engine_build; pointers are owned by the
 * engine and stay valid until the next build or destroy. */
typedef struct mcmi_device_csr {
    int64_t row_begin, row_end; /* global rows [row_begin, row_end) */
    int64_t nnz;
    int64_t* row_ptr;        /* [rows+1], starts at 0 */
    int64_t* col_idx;        /* [nnz] */
    double* values;          /* [nnz] */
    int64_t* chains_used;    /* [rows] */
    int64_t* entries_before; /* [rows] */
} mcmi_device_csr;

int mcmi_engine_create(int device, mcmi_engine** out, char* err, size_t errlen);
void mcmi_engine_destroy(mcmi_engine* e);
/* Builds rows [row_begin, row_end) of M from a device-resident B on `stream`
 * (a cudaStream_t; NULL = the engine's own stream).  Synchronises with the
 * stream once after the transition tables (the chain budget is derived on the
 * host with glibc log/ceil, mc_engine.cpp:12-33) and once at the end. */
int mcmi_engine_build(mcmi_engine* e, const mcmi_csr_view* b_dev, const mcmi_config* cfg,
                      int64_t row_begin, int64_t row_end, void* stream, mcmi_device_csr* out,
                      mcmi_stats* stats, char* err, size_t errlen);

/* Multi-GPU assembly over NVLink peer memory: stores this rank's
 * device shard (row_ptr [rows+1] starting at 0, col_idx / values [nnz]) into
 * each of `npeers` symmetric buffers laid out as
 *   [row_ptr: n_total+1 int64][col_idx: nnz_total int64][values: nnz_total f64]
 * (each array at a 16-byte boundary) at global rows [row_offset, row_offset+rows) and entries
 * [nnz_offset, nnz_offset+nnz) (row_ptr shifted by nnz_offset).  One kernel on
 * `stream`; the buffers are peer mappings (e.g. torch symmetric memory), the
 * caller barriers across ranks afterwards.  Replaces an NCCL all-gather-v of
 * the shards; rank order == row order gives the reference's assembly. */
int mcmi_scatter_shard(const int64_t* row_ptr, const int64_t* col_idx, const double* values, int64_t rows,
                       int64_t nnz, int64_t row_offset, int64_t nnz_offset, int64_t n_total, int64_t nnz_total,
                       void* const* peer_buffers, int npeers, void* stream);

/* ------------------------------------------------- consumer of M (§8f) */

/* SolverMethod / SolverConfig (solvers.hpp:11-18) */
#define MCMI_SOLVER_GMRES 0
#define MCMI_SOLVER_BICGSTAB 1

typedef struct mcmi_solver_config {
    int32_t method;   /* MCMI_SOLVER_*, default gmres */
    int32_t reserved;
    double rel_tol;   /* default 1e-6 */
    int64_t max_iters; /* default 30000 */
    int64_t restart;  /* GMRES only, default 50 */
} mcmi_solver_config;

/* SolveReport (solvers.hpp:20-30), without the history and x (x is an output buffer) */
typedef struct mcmi_solve_report {
    int32_t converged;
    int32_t breakdown;
    int64_t iterations;
    double final_rel_residual; /* true residual ||rhs - B x|| / ||rhs|| */
    double ms;                 /* device time */
} mcmi_solve_report;

void mcmi_solver_config_default(mcmi_solver_config* cfg);
/* Left-preconditioned GMRES / BiCGstab on device-resident B and M (M NULL =
 * unpreconditioned), mirroring solvers.cpp:54-238; rhs NULL means B * ones
 * (ones_product_rhs).  x: device buffer of n doubles (solution, x0 = 0). */
int mcmi_solve_device(const mcmi_csr_view* b_dev, const mcmi_csr_view* m_dev, const double* rhs_dev,
                      double* x_dev, const mcmi_solver_config* cfg, int device, void* stream,
                      mcmi_solve_report* rep, char* err, size_t errlen);

/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream): copies an
 * engine output into caller-owned host or device memory. */
int mcmi_copy(void* dst, const void* src, size_t bytes, void* stream);

/* Page-locks caller memory for this library's DMA (cudaHostRegister): host
 * buffers reused across mcmi_build_into calls should be registered once so
 * the device->host copies run asynchronously at full PCIe bandwidth. */
int mcmi_host_register(void* ptr, size_t bytes);
int mcmi_host_unregister(void* ptr);

/* ------------------------------- Matrix Market I/O and triplets (§8f rank 2) */

/* Host CSR owned by the library (parse / from_triplets output).  The arrays are
 * borrowed through mcmi_host_csr_get and stay valid until mcmi_host_csr_free. */
typedef struct mcmi_host_csr mcmi_host_csr;

/* mcspai::CsrMatrix::from_triplets (csr.cpp:17-58): sort by (row, col), sum
 * duplicates in the reference's sort order, prune exact zeros.  Errors:
 * MCMI_ERANGE "triplet index out of range".  rows/cols/vals hold `count`
 * entries (the reference's equal-length check lives in the caller's binding). */
int mcmi_from_triplets(int64_t n, const int64_t* rows, const int64_t* cols, const double* vals,
                       int64_t count, mcmi_host_csr** out, char* err, size_t errlen);
/* mcspai::parse_matrix_market (matrix_market.cpp:27-147) over `len` bytes of
 * text; MCMI_EPARSE errors carry the reference's "matrix market: line N: ..." */
int mcmi_mm_parse(const char* text, size_t len, mcmi_host_csr** out, char* err, size_t errlen);
/* mcspai::read_matrix_market_file (matrix_market.cpp:149-153) */
int mcmi_mm_read_file(const char* path, mcmi_host_csr** out, char* err, size_t errlen);
void mcmi_host_csr_get(const mcmi_host_csr* m, mcmi_csr_view* view);
void mcmi_host_csr_free(mcmi_host_csr* m);
/* mcspai::write_matrix_market (matrix_market.cpp:155-169): the same bytes
 * ("%lld %lld %.17g" lines).  buf == NULL: *len = bytes needed, MCMI_OK;
 * cap < needed: *len = needed, MCMI_ENOMEM. */
int mcmi_mm_format(const mcmi_csr_view* m, char* buf, size_t cap, size_t* len, char* err, size_t errlen);
/* mcspai::write_matrix_market_file (matrix_market.cpp:171-177) */
int mcmi_mm_write_file(const mcmi_csr_view* m, const char* path, char* err, size_t errlen);

/* ------------------------------------------------ recovery phase (§8f rank 4) */

/* mcspai::recover_inverse (recovery.hpp:22-23, recovery.cpp:7-33) on the GPU:
 * m is the dense row-major n x n B_hat^{-1} (host memory) and is replaced by
 * the recovered inverse, bit-identical to the reference.  s_diag / s_len are
 * RecoveryPlan::s_diag.  Errors: MCMI_EINVAL ("recovery plan length mismatch",
 * "tol must be positive"), MCMI_ERECOVERY ("singular update at row i"; m is
 * left unchanged). */
int mcmi_recover_inverse(double* m, int64_t n, const double* s_diag, int64_t s_len, double tol, int device,
                         char* err, size_t errlen);
/* The same on a device-resident matrix, in place, on `stream` (m_dev is left
 * partially updated on MCMI_ERECOVERY, like the reference's working copy). */
int mcmi_recover_inverse_device(double* m_dev, int64_t n, const double* s_diag, int64_t s_len, double tol,
                                int device, void* stream, char* err, size_t errlen);

/* Library identification: returns "mcmi <abi> sm_100a". */
const char* mcmi_version(void);

#ifdef __cplusplus
}
#endif
#endif
