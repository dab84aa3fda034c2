// kernels.cuh — internal interface between the host engine and the kernels.
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "mcmi.h"

namespace mcmi {

// Restores the calling thread's current CUDA device when a C-ABI entry point
// returns: the library switches devices internally (engines, shards), callers
// (PyTorch, a reference-side host program) must not see it.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Device-side scalar reductions and error slots of one build (zeroed per build).
struct Reductions {
    unsigned long long offmin_bits;  // min |b_ij| over off-diagonals (csr.cpp:88-105)
    unsigned long long offmax_bits;  // max |b_ij| over off-diagonals
    unsigned long long bnorm_bits;   // ||B_reduced||inf (csr.cpp:77-86)
    unsigned long long anorm_bits;   // ||A||inf (split.cpp:83-92)
    long long degenerate_row;        // first row with b_hat_ii == 0 (split.cpp:67-69), else LLONG_MAX
    long long bad_col_row;           // first row holding a column outside [0,n), else LLONG_MAX
    unsigned long long max_deg;      // max row length of A
    unsigned long long a_nnz;        // entries of A
    long long bad_rowptr_row;        // first row with an invalid row_ptr, else LLONG_MAX
};

// Transition tables (subsystem 1), one 32-byte record per state s:
//   rec[2s]   = {begin, deg, guide[0..3], guide[4..7]}
//   rec[2s+1] = {guide[8..11], guide[12..15], col (deg==1), guide scale ceil(deg/255)}
//   deg == 1 : rec[2s].zw holds the forced move's ratio (f64) instead of guide[0..7]
//   guide[m] (u8, in units of ceil(deg/255)) = first k with cum_k > m/16, so the
//   inverse-CDF scan for u starts at guide[floor(16u)] and returns the same k as
//   the reference's full scan (all skipped cum_k <= m/16 <= u).
//   ent[k]  = {cum_k, ratio_k}: running sequential sum of p (sample_transition's
//             `cum`, mc_engine.cpp:71-75) and a_k / p_k (mc_engine.cpp:94); the
//             last entry of a row with deg >= 2 stores cum = +inf, which makes
//             "first k with u < cum_k" return end-1 exactly when the reference's
//             scan falls through to its end-1 fallback (mc_engine.cpp:76), so the
//             device scan needs no bound or fallback
//   col[k]  = column of A (int32)
constexpr int kGuide = 16;

struct Tables {
    int64_t n;
    const uint4* rec;
    const double2* ent;
    const int* col;
    const double* b1_diag;  // diag(B_hat) = B1 (split.cpp:70)
    const unsigned char* tri;  // [n] L = 2 split-fold rows (k_tri_free), or nullptr
};

struct TableBuildArgs {
    int64_t n;
    const int64_t* row_ptr;
    const int64_t* col_idx;
    const double* values;
    double drop_fraction;
    int drop_mode;
    double alpha;
    int mode;
    // scratch / outputs
    Reductions* red;
    double* diag_val;     // [n]
    unsigned* a_cnt;      // [n]
    unsigned* a_off;      // [n+1]
    unsigned char* keep;  // [nnz] count-quantile keep flags (or nullptr)
    uint4* rec;           // [2n]
    double2* ent;
    int* col;
    double* b1_diag;
};

// Transition tables from a caller-built SplitSystem (mcmi_estimate_rows).
struct ApTableArgs {
    int64_t n;
    const int64_t* row_ptr;  // A's (and P's) row pointer
    const int64_t* col_idx;  // A's columns
    const double* a_values;
    const double* p_values;  // P on A's pattern
    Reductions* red;
    uint4* rec;
    double2* ent;
    int* col;
    double* b1_diag;
};

// The SplitSystem as matrices (mcmi_augment_and_split).
struct SplitExportArgs {
    int64_t n;
    const int64_t* row_ptr;
    const int64_t* col_idx;
    const double* values;
    double alpha;
    int mode;
    Reductions* red;
    double* diag_val;          // [n]
    unsigned char* has_diag;   // [n]
    int* bh_cnt;               // [n] b_hat row lengths
    int* a_cnt;                // [n] A row lengths
    double* b1_diag;           // [n]
    double* s_diag;            // [n]
    const int64_t* bh_row_ptr; // [n+1] (pass 1)
    const int64_t* a_row_ptr;  // [n+1] (pass 1)
    int64_t* bh_col;
    double* bh_val;
    int64_t* a_col;
    double* a_val;
    double* p_val;
};

// Walk + accumulate + per-row finalize (subsystems 2 and 3).
struct WalkArgs {
    Tables t;
    int64_t row_begin;      // global index of local row 0
    const int* row_list;    // nullptr: work item i is row row_begin + work_offset + i
    int64_t work_offset;
    int64_t n_work;
    int claim_rows;         // consecutive work items a warp claims at once (1 for row lists)
    int64_t n_chains, max_len;
    double delta;
    uint64_t seed;
    uint32_t rk[20];        // Philox round keys of `seed` (launch_walk fills them)
    int64_t retain_k;
    int rng_mode;
    int cap;                // hash capacity (power of two)
    int cap_limit;          // max distinct columns before the row overflows to the next tier
    int lanes;              // chains per batch (<= 32)
    int log_stride;         // max(max_len, 1) step deposits per chain
    unsigned log_magic;     // ceil(2^32 / log_stride) for log_stride >= 2: p / S == __umulhi(p, magic)
    int ell0;               // initial speculative draw stride (reference-stream mode)
    int log_n;              // launch_walk: round32(lanes * log_stride), deposit-log slots per warp
    int hash_shift;         // launch_walk: 32 - log2(cap)
    int log_shift;          // launch_walk: log2(log_stride) if a power of two, else -1
    long long warp_bytes;   // launch_walk: shared/global bytes per warp
    int deg_stats;          // count sum deg(s) (MCMI_FLAG_DEG_STATS)
    int unscaled;           // MCMI_FLAG_UNSCALED: rows of (I - A)^-1 (estimate_row), no scale / prune
    int nb_hint;            // L = 2: neighbourhood slot tables pay off (deposits per row >> 2-hop size)
    unsigned char* gscratch;  // global-tier per-warp accumulator + log (nullptr for smem tiers)
    // outputs, indexed by local row (row - row_begin)
    int* stage_col;
    double* stage_val;
    int64_t stage_base;     // offset of work item 0 in the staging pool
    int64_t stage_stride;   // entries per work item
    int* row_cnt;
    int64_t* row_src;
    int64_t* chains_used;
    int64_t* entries_before;
    unsigned long long* counters;  // [0] work cursor [1] steps [2] deg_sum [3] overflow count
    int* overflow_list;
};

cudaError_t launch_validate_row_ptr(const int64_t* row_ptr, int64_t n, int64_t nnz, Reductions* red,
                                   cudaStream_t s);
cudaError_t launch_table_build(const TableBuildArgs& a, int64_t nnz, bool drop_active,
                               cudaStream_t s);
cudaError_t launch_table_fill(const TableBuildArgs& a, cudaStream_t s);
cudaError_t launch_ap_tables(const ApTableArgs& a, cudaStream_t s);
cudaError_t launch_tri_free(const uint4* rec, const int* col, int64_t n, unsigned char* tri, cudaStream_t s);
// drop_small_entries: pass 0 row counts (value range first), pass 1 fill.
cudaError_t launch_drop_filter(const TableBuildArgs& a, bool drop_active, int pass, int* cnt, const int64_t* out_rp,
                               int64_t* oci, double* ov, cudaStream_t s);
// pass 0: norms, diagonal, row counts, ||A||; pass 1: fill b_hat / A / P.
cudaError_t launch_split_export(const SplitExportArgs& a, int pass, cudaStream_t s);
// pass 0: row counts into cnt; pass 1: fill with out_rp (exclusive scan of cnt).
cudaError_t launch_transition_probabilities(const int64_t* rp, const int64_t* ci, const double* v, int64_t n,
                                            int* cnt, const int64_t* out_rp, int64_t* out_ci, double* out_v,
                                            int pass, cudaStream_t s);
cudaError_t launch_count_quantile(const TableBuildArgs& a, int64_t nnz, int64_t n_drop,
                                  void* scratch, size_t scratch_bytes, cudaStream_t s);
size_t count_quantile_scratch_bytes(int64_t nnz);
// Global-tier walk kernels: __launch_bounds__(256, kGlMinBlocks), so up to
// 8 * kGlMinBlocks resident warps per SM (one accumulator table each).
#ifndef MCMI_GL_MINB
#define MCMI_GL_MINB 4
#endif
constexpr int kGlMinBlocks = MCMI_GL_MINB;
constexpr int kGlWarpsPerSm = 8 * kGlMinBlocks;
size_t walk_smem_bytes_per_warp(int cap, int lanes, int log_stride);
size_t walk_global_bytes_per_warp(int cap, int lanes, int log_stride);
cudaError_t launch_walk(const WalkArgs& a, int warps_per_block, int num_sms, bool global_tier,
                        int64_t max_warps, cudaStream_t s);

// retain_top_k / scale_columns over the rows of a CSR (rowops.cu).  top-k pass
// 0 writes per-row kept counts (int), pass 1 the kept entries at out_rp.
cudaError_t launch_topk_rows(const int64_t* rp, const int64_t* ci, const double* v, int64_t n, int64_t k,
                             const int64_t* diag, int pass, int* cnt, const int64_t* out_rp, int64_t* oci,
                             double* ov, cudaStream_t s);
cudaError_t launch_scale_columns(const int64_t* ci, const double* v, int64_t nnz, const double* b1, int64_t b1_len,
                                 double* out, int* bad, cudaStream_t s);

// Exclusive scans (assemble.cu).
size_t scan_scratch_bytes(int64_t n);
cudaError_t scan_u32_exclusive(const unsigned* in, unsigned* out, int64_t n, void* scratch,
                               cudaStream_t s);  // out[n] = total
cudaError_t scan_rows_exclusive(const int* in, int64_t* out, int64_t n, void* scratch,
                                cudaStream_t s);  // out[n] = total
cudaError_t launch_add_offset(int64_t* a, int64_t add, int64_t n, cudaStream_t s);
cudaError_t launch_compact(const int* stage_col, const double* stage_val, const int64_t* row_src,
                           const int* row_cnt, const int64_t* row_ptr, int64_t rows,
                           int64_t* col_out, double* val_out, cudaStream_t s);

// Recovery phase (recovery.cu): in-place recover_inverse on a device n x n
// row-major matrix; s_host = the plan's s_diag on the host.  *bad_row = the
// row of a singular update (MCMI_ERECOVERY) or -1.
int recover_device(double* m, int64_t n, const double* s_host, double tol, cudaStream_t st, int64_t* bad_row,
                   std::string& msg);

// Validation solvers on device (solver.cu).
int solve_device(const mcmi_csr_view& b, const mcmi_csr_view* m, const double* rhs, double* x,
                 const mcmi_solver_config& cfg, cudaStream_t s, mcmi_solve_report* rep, std::string& msg);

}  // namespace mcmi
