// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// the reference sources where they lie (/root/reference/proj/src/*.cpp) by
// oracle/Makefile into oracle/_ref/libmcspai_ref.so.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it.
//
// Every entry point forwards to one reference function:
//   ref_build          -> mcspai::compute_preconditioner / _serial  (mc_engine.hpp:80-86)
//   ref_split          -> mcspai::augment_and_split                 (split.hpp:34-35)
//   ref_drop           -> mcspai::drop_small_entries                (csr.hpp:76-77)
//   ref_budget         -> mcspai::derive_chain_budget               (mc_engine.hpp:55)
//   ref_estimate_row   -> mcspai::estimate_row                      (mc_engine.hpp:63-65)
//   ref_retain_top_k   -> mcspai::retain_top_k                      (mc_engine.hpp:70)
//   ref_rng_u32        -> mcspai::RngStream::next_u32               (rng.hpp:24-30)
//   ref_rng_double     -> mcspai::RngStream::next_double            (rng.hpp:39-41)
//   ref_gen            -> mcspai::make_* generators                 (synthetic.hpp:11-31)
//   ref_write_mm       -> mcspai::write_matrix_market_file          (matrix_market.hpp:24-25)
//   ref_read_mm        -> mcspai::read_matrix_market_file           (matrix_market.hpp:19-20)
//   ref_solve          -> mcspai::solve (gmres / bicgstab), rhs = B*1  (solvers.hpp:35-46)
// Exceptions are mapped to status codes: 1 invalid_argument, 2 SplitError,
// 3 out_of_range, 4 other.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "mcspai/csr.hpp"
#include "mcspai/dense_solve.hpp"
#include "mcspai/matrix_market.hpp"
#include "mcspai/recovery.hpp"
#include "mcspai/mc_engine.hpp"
#include "mcspai/solvers.hpp"
#include "mcspai/split.hpp"
#include "mcspai/synthetic.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace mcspai;

extern "C" {

// Mirrors mcspai::McConfig (mc_engine.hpp:15-26); same field layout as the
// product's mcmi_config prefix so one Python dict fills both.
struct ref_config {
    double epsilon;
    double delta;
    double alpha;
    int32_t mode;       // 0 plain, 1 sign_aware
    int32_t drop_mode;  // 0 value_range, 1 count_quantile
    double drop_fraction;
    int64_t retain_k;
    int32_t has_chains_override;
    int32_t has_max_len_override;
    int64_t chains_override;
    int64_t max_len_override;
    uint64_t master_seed;
};

}  // extern "C"

namespace {

McConfig to_cfg(const ref_config* c) {
    McConfig cfg;
    cfg.epsilon = c->epsilon;
    cfg.delta = c->delta;
    cfg.alpha = c->alpha;
    cfg.mode = c->mode == 0 ? AugmentationMode::plain : AugmentationMode::sign_aware;
    cfg.drop_mode = c->drop_mode == 0 ? DropMode::value_range : DropMode::count_quantile;
    cfg.drop_fraction = c->drop_fraction;
    cfg.retain_k = c->retain_k;
    if (c->has_chains_override) cfg.chains_override = c->chains_override;
    if (c->has_max_len_override) cfg.max_len_override = c->max_len_override;
    cfg.master_seed = c->master_seed;
    return cfg;
}

CsrMatrix to_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
    CsrMatrix m;
    m.n = n;
    m.row_ptr.assign(rp, rp + n + 1);
    const int64_t nnz = rp[n];
    m.col_idx.assign(ci, ci + nnz);
    m.values.assign(v, v + nnz);
    return m;
}

int fail(const std::exception& e, int code, char* err, size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

template <class F>
int guarded(F&& f, char* err, size_t errlen) {
    try {
        f();
        return 0;
    } catch (const SplitError& e) {
        return fail(e, 2, err, errlen);
    } catch (const std::invalid_argument& e) {
        return fail(e, 1, err, errlen);
    } catch (const std::out_of_range& e) {
        return fail(e, 3, err, errlen);
    } catch (const std::exception& e) {
        return fail(e, 4, err, errlen);
    }
}

void copy_csr(const CsrMatrix& m, int64_t* rp, int64_t* ci, double* v) {
    if (rp) std::memcpy(rp, m.row_ptr.data(), sizeof(int64_t) * (m.n + 1));
    if (ci) std::memcpy(ci, m.col_idx.data(), sizeof(int64_t) * m.nnz());
    if (v) std::memcpy(v, m.values.data(), sizeof(double) * m.nnz());
}

}  // namespace

extern "C" {

int ref_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// ---- compute_preconditioner ------------------------------------------------
// seconds (may be NULL) receives the wall time of the reference call alone:
// the CsrMatrix is built before the clock starts, as a reference caller holds
// one already (bench.py --impl reference times exactly this).
int ref_build_timed(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                    const ref_config* c, int n_threads, int serial, void** out,
                    double* seconds, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] {
            const CsrMatrix b = to_csr(n, rp, ci, v);
            const McConfig cfg = to_cfg(c);
            const auto t0 = std::chrono::steady_clock::now();
            auto res = std::make_unique<ApproxInverse>(
                serial ? compute_preconditioner_serial(b, cfg)
                       : compute_preconditioner(b, cfg, n_threads));
            const auto t1 = std::chrono::steady_clock::now();
            if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
            *out = res.release();
        },
        err, errlen);
}

int ref_build(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              const ref_config* c, int n_threads, int serial, void** out,
              char* err, size_t errlen) {
    return ref_build_timed(n, rp, ci, v, c, n_threads, serial, out, nullptr, err, errlen);
}

void ref_result_sizes(const void* h, int64_t* n, int64_t* nnz) {
    const auto* r = static_cast<const ApproxInverse*>(h);
    *n = r->m.n;
    *nnz = r->m.nnz();
}

void ref_result_copy(const void* h, int64_t* rp, int64_t* ci, double* v,
                     int64_t* chains_used, int64_t* entries_before,
                     int64_t* n_chains, int64_t* max_len) {
    const auto* r = static_cast<const ApproxInverse*>(h);
    copy_csr(r->m, rp, ci, v);
    for (int64_t i = 0; i < r->m.n; ++i) {
        if (chains_used) chains_used[i] = r->row_meta[i].chains_used;
        if (entries_before) entries_before[i] = r->row_meta[i].entries_before_retention;
    }
    if (n_chains) *n_chains = r->budget_echo.n_chains;
    if (max_len) *max_len = r->budget_echo.max_len;
}

int ref_result_write_mm(const void* h, const char* path, char* err, size_t errlen) {
    const auto* r = static_cast<const ApproxInverse*>(h);
    return guarded([&] { write_matrix_market_file(r->m, path); }, err, errlen);
}

void ref_result_free(void* h) { delete static_cast<ApproxInverse*>(h); }

// ---- CSR handles (generators, drop, MM I/O) ---------------------------------
void ref_csr_sizes(const void* h, int64_t* n, int64_t* nnz) {
    const auto* m = static_cast<const CsrMatrix*>(h);
    *n = m->n;
    *nnz = m->nnz();
}

void ref_csr_copy(const void* h, int64_t* rp, int64_t* ci, double* v) {
    copy_csr(*static_cast<const CsrMatrix*>(h), rp, ci, v);
}

void ref_csr_free(void* h) { delete static_cast<CsrMatrix*>(h); }

// kind: 0 tridiagonal(a), 1 convection_diffusion(a, x, y), 2 brusselator(a),
//       3 random_ddm(a, fill=x, seed), 4 broad_spectrum(a, nnz_per_row=(int)x, lo=y, hi=z, seed)
void* ref_gen(int kind, int64_t a, double x, double y, double z, uint64_t seed) {
    CsrMatrix m;
    switch (kind) {
        case 0: m = make_tridiagonal(a); break;
        case 1: m = make_convection_diffusion(a, x, y); break;
        case 2: m = make_brusselator(a); break;
        case 3: m = make_random_ddm(a, x, seed); break;
        case 4: m = make_broad_spectrum(a, static_cast<index_t>(x), y, z, seed); break;
        default: return nullptr;
    }
    return new CsrMatrix(std::move(m));
}

int ref_write_mm(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                 const char* path, char* err, size_t errlen) {
    return guarded([&] { write_matrix_market_file(to_csr(n, rp, ci, v), path); },
                   err, errlen);
}

int ref_read_mm(const char* path, void** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] { *out = new CsrMatrix(read_matrix_market_file(path)); }, err,
        errlen);
}

// parse_matrix_market over an in-memory text (std::istringstream, as the
// reference's own tests do)
int ref_parse_mm(const char* text, size_t len, void** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] {
            std::istringstream in(std::string(text, len));
            *out = new CsrMatrix(parse_matrix_market(in));
        },
        err, errlen);
}

// write_matrix_market into a std::ostringstream; returns a malloc'd buffer
char* ref_format_mm(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, size_t* len) {
    std::ostringstream out;
    write_matrix_market(to_csr(n, rp, ci, v), out);
    const std::string s = out.str();
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
    *len = s.size();
    return buf;
}

void ref_free_buf(char* p) { std::free(p); }

// recover_inverse (recovery.cpp:7-33): out = recovered n x n (row-major);
// status 5 = RecoveryError, 1 = invalid_argument
int ref_recover(int64_t n, const double* m, const double* s, int64_t s_len, double tol, double* out,
                char* err, size_t errlen) {
    try {
        DenseMatrix d(n);
        std::memcpy(d.values.data(), m, sizeof(double) * n * n);
        RecoveryPlan plan{std::vector<double>(s, s + s_len)};
        const DenseMatrix r = recover_inverse(d, plan, tol);
        std::memcpy(out, r.values.data(), sizeof(double) * n * n);
        return 0;
    } catch (const RecoveryError& e) {
        return fail(e, 5, err, errlen);
    } catch (const std::invalid_argument& e) {
        return fail(e, 1, err, errlen);
    }
}

// dense_inverse (dense_solve.cpp) — produces B_hat^{-1} inputs like the reference tests
int ref_dense_inverse(int64_t n, const double* m, double* out, char* err, size_t errlen) {
    return guarded(
        [&] {
            DenseMatrix d(n);
            std::memcpy(d.values.data(), m, sizeof(double) * n * n);
            const DenseMatrix r = dense_inverse(d);
            std::memcpy(out, r.values.data(), sizeof(double) * n * n);
        },
        err, errlen);
}

int ref_from_triplets(int64_t n, const int64_t* r, const int64_t* c, const double* v, int64_t m,
                      void** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] {
            *out = new CsrMatrix(CsrMatrix::from_triplets(
                n, std::vector<index_t>(r, r + m), std::vector<index_t>(c, c + m),
                std::vector<double>(v, v + m)));
        },
        err, errlen);
}

int ref_drop(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
             double p, int drop_mode, void** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] {
            *out = new CsrMatrix(drop_small_entries(
                to_csr(n, rp, ci, v), p,
                drop_mode == 0 ? DropMode::value_range : DropMode::count_quantile));
        },
        err, errlen);
}

// ---- split ------------------------------------------------------------------
int ref_split(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              double alpha, int mode, void** out, char* err, size_t errlen) {
    *out = nullptr;
    return guarded(
        [&] {
            *out = new SplitSystem(augment_and_split(
                to_csr(n, rp, ci, v), alpha,
                mode == 0 ? AugmentationMode::plain : AugmentationMode::sign_aware));
        },
        err, errlen);
}

// A caller-built SplitSystem (the reference's own tests build one by hand,
// test_mc_engine.cpp:112-127): a = (rp, ci, av), p = A's pattern with pv.
void* ref_split_from_ap(int64_t n, const int64_t* rp, const int64_t* ci, const double* av, const double* pv) {
    auto* s = new SplitSystem();
    s->a = to_csr(n, rp, ci, av);
    s->p = to_csr(n, rp, ci, pv);
    s->b1_diag.assign(static_cast<size_t>(n), 1.0);
    s->s_diag.assign(static_cast<size_t>(n), 0.0);
    s->a_norm = 0.5;
    return s;
}

// which: 0 b_hat, 1 a, 2 p
const void* ref_split_matrix(const void* h, int which) {
    const auto* s = static_cast<const SplitSystem*>(h);
    return which == 0 ? &s->b_hat : which == 1 ? &s->a : &s->p;
}

void ref_split_diag(const void* h, double* b1_diag, double* s_diag, double* a_norm) {
    const auto* s = static_cast<const SplitSystem*>(h);
    if (b1_diag) std::memcpy(b1_diag, s->b1_diag.data(), sizeof(double) * s->a.n);
    if (s_diag) std::memcpy(s_diag, s->s_diag.data(), sizeof(double) * s->a.n);
    if (a_norm) *a_norm = s->a_norm;
}

void ref_split_free(void* h) { delete static_cast<SplitSystem*>(h); }

// ---- budget, estimate_row, retain_top_k ---------------------------------------
int ref_budget(const ref_config* c, double a_norm, int64_t* n_chains, int64_t* max_len,
               char* err, size_t errlen) {
    return guarded(
        [&] {
            const ChainBudget b = derive_chain_budget(to_cfg(c), a_norm);
            *n_chains = b.n_chains;
            *max_len = b.max_len;
        },
        err, errlen);
}

// Returns the row length; copies up to cap entries.
int64_t ref_estimate_row(const void* split, int64_t r, int64_t n_chains, int64_t max_len,
                         double delta, uint64_t seed, int64_t* cols, double* vals,
                         int64_t cap) {
    const auto* s = static_cast<const SplitSystem*>(split);
    const SparseRow row =
        estimate_row(*s, r, ChainBudget{n_chains, max_len}, delta, RngStream(seed, r));
    for (int64_t i = 0; i < static_cast<int64_t>(row.size()) && i < cap; ++i) {
        cols[i] = row[i].first;
        vals[i] = row[i].second;
    }
    return static_cast<int64_t>(row.size());
}

int64_t ref_retain_top_k(int64_t len, int64_t* cols, double* vals, int64_t k,
                         int64_t diag_col) {
    SparseRow row;
    for (int64_t i = 0; i < len; ++i) row.emplace_back(cols[i], vals[i]);
    const SparseRow kept = retain_top_k(std::move(row), k, diag_col);
    for (std::size_t i = 0; i < kept.size(); ++i) {
        cols[i] = kept[i].first;
        vals[i] = kept[i].second;
    }
    return static_cast<int64_t>(kept.size());
}

// ---- validation solvers (the consumer of M; iteration-count parity tier) ----
// method 0 gmres, 1 bicgstab; precond may be null (n_m < 0).  rhs = B * ones.
int ref_solve(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t n_m,
              const int64_t* mrp, const int64_t* mci, const double* mv, int method,
              double rel_tol, int64_t max_iters, int64_t restart, int64_t* iterations,
              int* converged, double* final_rel_residual, char* err, size_t errlen) {
    return guarded(
        [&] {
            const CsrMatrix b = to_csr(n, rp, ci, v);
            CsrMatrix m;
            if (n_m >= 0) m = to_csr(n_m, mrp, mci, mv);
            SolverConfig cfg;
            cfg.method = method == 0 ? SolverMethod::gmres : SolverMethod::bicgstab;
            cfg.rel_tol = rel_tol;
            cfg.max_iters = max_iters;
            cfg.restart = restart;
            const SolveReport r = solve(b, ones_product_rhs(b), n_m >= 0 ? &m : nullptr, cfg);
            *iterations = r.iterations;
            *converged = r.converged ? 1 : 0;
            *final_rel_residual = r.final_rel_residual;
        },
        err, errlen);
}

// ---- RNG ----------------------------------------------------------------------
void ref_rng_u32(uint64_t seed, uint64_t id, int64_t count, uint32_t* out) {
    RngStream s(seed, id);
    for (int64_t i = 0; i < count; ++i) out[i] = s.next_u32();
}

void ref_rng_double(uint64_t seed, uint64_t id, int64_t count, double* out) {
    RngStream s(seed, id);
    for (int64_t i = 0; i < count; ++i) out[i] = s.next_double();
}

}  // extern "C"
