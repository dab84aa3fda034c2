// include/mcmi/mcspai_compat.hpp — header-only C++ drop-in over the C-ABI.
//
// Replaces the body of
//   mcspai::compute_preconditioner(const CsrMatrix&, const McConfig&, int)
//   (/root/reference/proj/include/mcspai/mc_engine.hpp:80-81,
//    /root/reference/proj/src/mc_engine.cpp:230-233)
// with the B200 build, operating directly on the reference's own types:
//
//   #include "mcmi/mcspai_compat.hpp"
//   ApproxInverse compute_preconditioner(const CsrMatrix& b, const McConfig& cfg, int) {
//       return mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(b, cfg);
//   }
//
// The templates only touch the fields the reference declares:
//   CsrMatrix      n, row_ptr, col_idx, values          (csr.hpp:16-21)
//   McConfig       epsilon .. master_seed                (mc_engine.hpp:15-26)
//   ApproxInverse  m, row_meta, config_echo, budget_echo, seed_echo (mc_engine.hpp:39-45)
// Errors are re-thrown as the reference throws them: std::invalid_argument
// (csr.cpp:129, split.cpp:48, mc_engine.cpp:14), SplitErrorT (split.cpp:68,95),
// std::out_of_range (bad column index), std::runtime_error (CUDA / device).
//
// §8f rank 2, the formats either side of the build (same results byte for byte):
//   from_triplets<CsrMatrix>(n, rows, cols, vals)            csr.cpp:17-58
//   parse_matrix_market<CsrMatrix, ParseError>(istream&)     matrix_market.cpp:27-147
//   read_matrix_market_file<CsrMatrix, ParseError>(path)     matrix_market.cpp:149-153
//   write_matrix_market(m, ostream&)                         matrix_market.cpp:155-169
//   write_matrix_market_file(m, path)                        matrix_market.cpp:171-177
// §8f rank 4:
//   recover_inverse<DenseMatrix, RecoveryError>(m, plan, tol) recovery.cpp:7-33
#ifndef MCMI_MCSPAI_COMPAT_HPP
#define MCMI_MCSPAI_COMPAT_HPP

#include <chrono>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <istream>
#include <iterator>
#include <ostream>
#include <new>
#include <stdexcept>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#ifdef __linux__
#include <sys/mman.h>
#endif

#include "../mcmi.h"

namespace mcmi {
namespace compat {

struct Options {
    int device = 0;                      // CUDA device ordinal
    int rng_mode = MCMI_RNG_REFERENCE;   // byte-identical to the reference by default
    int n_gpus = 0;                      // row blocks on devices device..device+n_gpus-1; 0 = env MCMI_GPUS or 1
};

template <class CfgT>
mcmi_config to_config(const CfgT& cfg, const Options& opt) {
    mcmi_config c;
    mcmi_config_default(&c);
    c.epsilon = cfg.epsilon;
    c.delta = cfg.delta;
    c.alpha = cfg.alpha;
    c.mode = static_cast<int32_t>(cfg.mode);            // plain = 0, sign_aware = 1
    c.drop_mode = static_cast<int32_t>(cfg.drop_mode);  // value_range = 0, count_quantile = 1
    c.drop_fraction = cfg.drop_fraction;
    c.retain_k = static_cast<int64_t>(cfg.retain_k);
    c.has_chains_override = cfg.chains_override.has_value() ? 1 : 0;
    c.chains_override = cfg.chains_override.value_or(0);
    c.has_max_len_override = cfg.max_len_override.has_value() ? 1 : 0;
    c.max_len_override = cfg.max_len_override.value_or(0);
    c.master_seed = cfg.master_seed;
    c.rng_mode = opt.rng_mode;
    c.device = opt.device;
    c.n_gpus = opt.n_gpus;
    return c;
}

template <class SplitErrorT>
[[noreturn]] inline void rethrow(int code, const char* msg) {
    switch (code) {
        case MCMI_EINVAL: throw std::invalid_argument(msg);
        case MCMI_ESPLIT: throw SplitErrorT(msg);
        case MCMI_ERANGE: throw std::out_of_range(msg);
        case MCMI_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(std::string("mcmi: ") + msg);
    }
}

namespace detail {

// Sizing of the result's entry vectors while the GPU walks.  First-touching
// fresh memory is the host's bottleneck (tools/host_probe.cu on the B200 box:
// ~12.5 GB/s of page faults, 2 MB pages included; C2's two 1.28 GB vectors
// take ~200 ms), so it starts with the build: each vector reserves a generous
// virtual range (nothing touched), asks for 2 MB pages, and grows by
// value-initialising resizes up to the current limit (16M entries until the
// library's estimate is known, then the estimate), publishing its ready size;
// the ready prefix is attached to the job, whose copier fills it as row chunks
// land.  The data pointer never moves while size <= the reserved capacity.
struct Presizer {
    std::mutex mu;
    std::condition_variable cv;
    int64_t limit = int64_t{16} << 20;
    bool limit_final = false, stop = false;
    int64_t ready[2] = {0, 0};
};

template <class VecT>
void reserve_huge(VecT& v, size_t count) {
    v.reserve(count);
#ifdef __linux__
    const size_t bytes = count * sizeof(typename VecT::value_type);
    if (bytes >= (size_t{4} << 20)) {
        const uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + 4095) & ~uintptr_t(4095);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(v.data()) + bytes) & ~uintptr_t(4095);
        if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
    }
#endif
}

template <class VecT, class Publish, class Refresh>
void grow_within(VecT& v, size_t reserved, int k, Presizer& p, Publish&& publish, Refresh&& refresh) {
    const size_t step = size_t{16} << 20;  // 128 MB of entries per resize
    for (;;) {
        size_t target;
        {
            std::unique_lock<std::mutex> lk(p.mu);
            for (;;) {
                const size_t lim = static_cast<size_t>(std::min<int64_t>(p.limit, reserved));
                if (p.stop) return;
                if (v.size() < lim) {
                    target = std::min(lim, v.size() + step);
                    break;
                }
                if (p.limit_final) {  // caught up: poll the library's refreshed estimate
                    lk.unlock();
                    const int64_t e = refresh();
                    lk.lock();
                    if (e > p.limit) {
                        p.limit = e;
                        continue;
                    }
                }
                p.cv.wait_for(lk, std::chrono::milliseconds(2));
            }
        }
        v.resize(target);
        publish(k, static_cast<int64_t>(target));
    }
}

}  // namespace detail

// The reference's compute_preconditioner on the B200 build.  The build runs on
// a library thread (mcmi_build_start) and streams M into page-locked memory
// chunk by chunk.  Meanwhile two host threads grow the result's std::vectors
// (detail::grow_within, sized by the library's early estimate,
// mcmi_job_estimate) and attach their ready prefix to the job
// (mcmi_job_attach), whose copier moves each landed chunk into them; only what
// is left when the build ends is copied afterwards.  An estimate that falls
// short just costs a regrow; the result never depends on it.
template <class ApproxInverseT, class SplitErrorT, class CsrT, class CfgT>
ApproxInverseT compute_preconditioner(const CsrT& b, const CfgT& cfg, const Options& opt = {}) {
    const mcmi_config c = to_config(cfg, opt);
    const mcmi_csr_view view{static_cast<int64_t>(b.n),
                             reinterpret_cast<const int64_t*>(b.row_ptr.data()),
                             reinterpret_cast<const int64_t*>(b.col_idx.data()), b.values.data()};
    char err[512] = {0};
    // MCMI_COMPAT_TRACE=1: phase timestamps of this call on stderr (tuning)
    static const bool trace = std::getenv("MCMI_COMPAT_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (trace)
            std::fprintf(stderr, "mcmi compat: %-10s %8.2f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    mcmi_job* job = nullptr;
    int code = mcmi_build_start(&view, &c, 0, -1, &job, err, sizeof err);
    if (code != MCMI_OK) rethrow<SplitErrorT>(code, err);
    ApproxInverseT out;
    const int64_t nnz_b = b.n > 0 ? static_cast<int64_t>(b.row_ptr[b.n]) : 0;
    const size_t reserved = static_cast<size_t>(std::min<int64_t>(std::max<int64_t>(nnz_b * 16, 1 << 20), int64_t{1} << 31));
    detail::Presizer ps;
    // until the estimate arrives, grow to nnz(B) entries: M holds every row's
    // diagonal and, for any budget worth a GPU, more than B's pattern
    ps.limit = std::max<int64_t>(ps.limit, std::min<int64_t>(nnz_b, static_cast<int64_t>(reserved)));
    int64_t* col_ptr = nullptr;  // stable: the vectors never outgrow `reserved` while attached
    double* val_ptr = nullptr;
    auto publish = [&](int k, int64_t ready) {
        std::lock_guard<std::mutex> lk(ps.mu);
        ps.ready[k] = ready;
        const int64_t both = std::min(ps.ready[0], ps.ready[1]);
        if (both > 0) mcmi_job_attach(job, col_ptr, val_ptr, both);
    };
    auto refresh = [&] {  // the library's latest (never lowered) estimate
        int64_t e = -1;
        return mcmi_job_estimate(job, &e) == MCMI_OK ? e : int64_t{-1};
    };
    std::thread sizers[2];
    try {
        detail::reserve_huge(out.m.col_idx, reserved);
        detail::reserve_huge(out.m.values, reserved);
        col_ptr = reinterpret_cast<int64_t*>(out.m.col_idx.data());
        val_ptr = out.m.values.data();
        sizers[0] = std::thread([&] { detail::grow_within(out.m.col_idx, reserved, 0, ps, publish, refresh); });
        sizers[1] = std::thread([&] { detail::grow_within(out.m.values, reserved, 1, ps, publish, refresh); });
    } catch (...) {  // no memory or no thread: the vectors are sized after the build
    }
    auto stop_sizers = [&] {
        {
            std::lock_guard<std::mutex> lk(ps.mu);
            ps.stop = true;
        }
        ps.cv.notify_all();
        for (auto& t : sizers)
            if (t.joinable()) t.join();
    };
    int64_t est = -1;
    const int est_code = mcmi_job_estimate(job, &est);
    {
        std::lock_guard<std::mutex> lk(ps.mu);
        ps.limit = (est_code == MCMI_OK && est > 0) ? est : 0;
        ps.limit_final = true;
    }
    ps.cv.notify_all();
    mark("estimate");
    const int64_t rows = b.n > 0 ? static_cast<int64_t>(b.n) : 0;
    try {
        detail::reserve_huge(out.m.row_ptr, static_cast<size_t>(rows) + 1);
        detail::reserve_huge(out.row_meta, static_cast<size_t>(rows));
        out.m.row_ptr.resize(static_cast<size_t>(rows) + 1);
        out.row_meta.resize(static_cast<size_t>(rows));
    } catch (...) {
        stop_sizers();
        mcmi_job_finish(job, nullptr, nullptr, nullptr, 0);
        throw;
    }
    mark("meta sized");
    mcmi_result* res = nullptr;
    int64_t delivered = 0;
    code = mcmi_job_finish(job, &res, &delivered, err, sizeof err);
    mark("built");
    stop_sizers();
    mark("presized");
    if (code != MCMI_OK) rethrow<SplitErrorT>(code, err);
    struct Guard {
        mcmi_result* r;
        ~Guard() { mcmi_result_free(r); }
    } guard{res};
    int64_t n = 0, nnz = 0;
    mcmi_result_sizes(res, &n, &nnz);
    out.m.n = n;
    out.m.row_ptr.resize(static_cast<size_t>(n) + 1);
    out.m.col_idx.resize(static_cast<size_t>(nnz));  // shrinks in place, or grows keeping the delivered prefix
    out.m.values.resize(static_cast<size_t>(nnz));
    delivered = std::min(delivered, nnz);
    int64_t n_chains = 0, max_len = 0;
    if (mcmi_result_copy(res, reinterpret_cast<int64_t*>(out.m.row_ptr.data()), nullptr, nullptr, nullptr, nullptr,
                         &n_chains, &max_len) != MCMI_OK ||
        mcmi_result_copy_range(res, delivered, nnz, reinterpret_cast<int64_t*>(out.m.col_idx.data()),
                               out.m.values.data()) != MCMI_OK)
        throw std::runtime_error("mcmi: result copy failed");
    mark("copied");
    if (trace) std::fprintf(stderr, "mcmi compat: delivered %lld of %lld entries early\n",
                            static_cast<long long>(delivered), static_cast<long long>(nnz));
    out.row_meta.resize(static_cast<size_t>(n));
    const int64_t *chains = nullptr, *before = nullptr;  // RowMeta straight from the result's arrays
    mcmi_result_view(res, nullptr, nullptr, nullptr, &chains, &before);
    for (int64_t i = 0; i < n; ++i) {
        out.row_meta[i].chains_used = chains[i];
        out.row_meta[i].entries_before_retention = before[i];
    }
    out.config_echo = cfg;
    out.budget_echo.n_chains = n_chains;
    out.budget_echo.max_len = max_len;
    out.seed_echo = cfg.master_seed;
    mark("done");
    return out;
}

namespace detail {

template <class CsrT>
mcmi_csr_view view_of(const CsrT& m) {
    return mcmi_csr_view{static_cast<int64_t>(m.n), reinterpret_cast<const int64_t*>(m.row_ptr.data()),
                         reinterpret_cast<const int64_t*>(m.col_idx.data()), m.values.data()};
}

template <class CsrT>
CsrT take(mcmi_host_csr* h) {
    mcmi_csr_view v;
    mcmi_host_csr_get(h, &v);
    CsrT m;
    m.n = v.n;
    const int64_t nnz = v.n > 0 ? v.row_ptr[v.n] : 0;
    m.row_ptr.assign(v.row_ptr, v.row_ptr + (v.n > 0 ? v.n + 1 : 0));
    if (v.n <= 0) m.row_ptr.assign(1, 0);
    m.col_idx.assign(v.col_idx, v.col_idx + nnz);
    m.values.assign(v.values, v.values + nnz);
    mcmi_host_csr_free(h);
    return m;
}

template <class ParseErrorT>
[[noreturn]] inline void rethrow_io(int code, const char* msg) {
    switch (code) {
        case MCMI_EPARSE: throw ParseErrorT(msg);
        case MCMI_EINVAL: throw std::invalid_argument(msg);
        case MCMI_ERANGE: throw std::out_of_range(msg);
        case MCMI_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

}  // namespace detail

template <class CsrT, class IndexVec, class ValueVec>
CsrT from_triplets(int64_t n, const IndexVec& rows, const IndexVec& cols, const ValueVec& vals) {
    if (rows.size() != cols.size() || rows.size() != vals.size())  // csr.cpp:20-21
        throw std::invalid_argument("triplet arrays must have equal length");
    char err[512] = {0};
    mcmi_host_csr* h = nullptr;
    const int code = mcmi_from_triplets(n, reinterpret_cast<const int64_t*>(rows.data()),
                                        reinterpret_cast<const int64_t*>(cols.data()), vals.data(),
                                        static_cast<int64_t>(rows.size()), &h, err, sizeof err);
    if (code != MCMI_OK) detail::rethrow_io<std::runtime_error>(code, err);
    return detail::take<CsrT>(h);
}

template <class CsrT, class ParseErrorT>
CsrT parse_matrix_market(std::istream& in) {
    const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    char err[512] = {0};
    mcmi_host_csr* h = nullptr;
    const int code = mcmi_mm_parse(text.data(), text.size(), &h, err, sizeof err);
    if (code != MCMI_OK) detail::rethrow_io<ParseErrorT>(code, err);
    return detail::take<CsrT>(h);
}

template <class CsrT, class ParseErrorT>
CsrT read_matrix_market_file(const std::string& path) {
    char err[512] = {0};
    mcmi_host_csr* h = nullptr;
    const int code = mcmi_mm_read_file(path.c_str(), &h, err, sizeof err);
    if (code != MCMI_OK) detail::rethrow_io<ParseErrorT>(code, err);
    return detail::take<CsrT>(h);
}

template <class CsrT>
void write_matrix_market(const CsrT& m, std::ostream& out) {
    const mcmi_csr_view v = detail::view_of(m);
    char err[512] = {0};
    size_t len = 0;
    std::string buf(static_cast<size_t>(128 + 48 * m.values.size()), '\0');
    int code = mcmi_mm_format(&v, buf.data(), buf.size(), &len, err, sizeof err);
    if (code == MCMI_ENOMEM && len > buf.size()) {
        buf.resize(len);
        code = mcmi_mm_format(&v, buf.data(), buf.size(), &len, err, sizeof err);
    }
    if (code != MCMI_OK) detail::rethrow_io<std::runtime_error>(code, err);
    out.write(buf.data(), static_cast<std::streamsize>(len));
    if (!out) throw std::runtime_error("matrix market: write failure");
}

template <class CsrT>
void write_matrix_market_file(const CsrT& m, const std::string& path) {
    const mcmi_csr_view v = detail::view_of(m);
    char err[512] = {0};
    const int code = mcmi_mm_write_file(&v, path.c_str(), err, sizeof err);
    if (code != MCMI_OK) detail::rethrow_io<std::runtime_error>(code, err);
}

template <class DenseT, class RecoveryErrorT, class PlanT>
DenseT recover_inverse(const DenseT& b_hat_inv, const PlanT& plan, double tol = 1e-12, const Options& opt = {}) {
    DenseT out = b_hat_inv;
    char err[512] = {0};
    const int code = mcmi_recover_inverse(out.values.data(), static_cast<int64_t>(out.n), plan.s_diag.data(),
                                          static_cast<int64_t>(plan.s_diag.size()), tol, opt.device, err, sizeof err);
    if (code == MCMI_ERECOVERY) throw RecoveryErrorT(err);
    if (code != MCMI_OK) detail::rethrow_io<std::runtime_error>(code, err);
    return out;
}

// ---- fine-grained building blocks on the reference's types

template <class ChainBudgetT, class CfgT>
ChainBudgetT derive_chain_budget(const CfgT& cfg, double a_norm) {  // mc_engine.hpp:55
    const mcmi_config c = to_config(cfg, Options{});
    char err[256] = {0};
    int64_t nc = 0, ml = 0;
    const int code = mcmi_derive_chain_budget(&c, a_norm, &nc, &ml, err, sizeof err);
    if (code != MCMI_OK) rethrow<std::runtime_error>(code, err);
    ChainBudgetT b;
    b.n_chains = nc;
    b.max_len = ml;
    return b;
}

template <class CsrT, class ModeT>
CsrT drop_small_entries(const CsrT& m, double p, ModeT mode, const Options& opt = {}) {  // csr.hpp:76-77
    const mcmi_csr_view v = detail::view_of(m);
    CsrT out;
    out.n = m.n;
    out.row_ptr.resize(static_cast<size_t>(m.n) + 1);
    out.col_idx.resize(m.col_idx.size());
    out.values.resize(m.values.size());
    char err[512] = {0};
    int64_t nnz = 0;
    const int code = mcmi_drop_small_entries(&v, p, static_cast<int32_t>(mode), opt.device,
                                             reinterpret_cast<int64_t*>(out.row_ptr.data()),
                                             reinterpret_cast<int64_t*>(out.col_idx.data()), out.values.data(), &nnz,
                                             err, sizeof err);
    if (code != MCMI_OK) rethrow<std::runtime_error>(code, err);
    out.col_idx.resize(static_cast<size_t>(nnz));
    out.values.resize(static_cast<size_t>(nnz));
    return out;
}

template <class CsrT>
CsrT transition_probabilities(const CsrT& a, const Options& opt = {}) {  // split.hpp:39
    const mcmi_csr_view v = detail::view_of(a);
    CsrT out;
    out.n = a.n;
    out.row_ptr.resize(static_cast<size_t>(a.n) + 1);
    out.col_idx.resize(a.col_idx.size());
    out.values.resize(a.values.size());
    char err[512] = {0};
    int64_t nnz = 0;
    const int code = mcmi_transition_probabilities(&v, opt.device, reinterpret_cast<int64_t*>(out.row_ptr.data()),
                                                   reinterpret_cast<int64_t*>(out.col_idx.data()), out.values.data(),
                                                   &nnz, err, sizeof err);
    if (code != MCMI_OK) rethrow<std::runtime_error>(code, err);
    out.col_idx.resize(static_cast<size_t>(nnz));
    out.values.resize(static_cast<size_t>(nnz));
    return out;
}

template <class SplitSystemT, class SplitErrorT, class CsrT, class ModeT>
SplitSystemT augment_and_split(const CsrT& b, double alpha, ModeT mode, const Options& opt = {}) {  // split.hpp:34-35
    const mcmi_csr_view v = detail::view_of(b);
    char err[512] = {0};
    mcmi_split_system* h = nullptr;
    const int code = mcmi_augment_and_split(&v, alpha, static_cast<int32_t>(mode), opt.device, &h, err, sizeof err);
    if (code != MCMI_OK) rethrow<SplitErrorT>(code, err);
    struct Guard {
        mcmi_split_system* h;
        ~Guard() { mcmi_split_free(h); }
    } guard{h};
    int64_t n = 0, nb = 0, na = 0;
    double a_norm = 0.0;
    mcmi_split_sizes(h, &n, &nb, &na, &a_norm);
    SplitSystemT s;
    s.b_hat.n = s.a.n = s.p.n = n;
    s.b_hat.row_ptr.resize(static_cast<size_t>(n) + 1);
    s.b_hat.col_idx.resize(static_cast<size_t>(nb));
    s.b_hat.values.resize(static_cast<size_t>(nb));
    s.a.row_ptr.resize(static_cast<size_t>(n) + 1);
    s.a.col_idx.resize(static_cast<size_t>(na));
    s.a.values.resize(static_cast<size_t>(na));
    s.p.values.resize(static_cast<size_t>(na));
    s.b1_diag.resize(static_cast<size_t>(n));
    s.s_diag.resize(static_cast<size_t>(n));
    mcmi_split_copy(h, reinterpret_cast<int64_t*>(s.b_hat.row_ptr.data()),
                    reinterpret_cast<int64_t*>(s.b_hat.col_idx.data()), s.b_hat.values.data(), s.b1_diag.data(),
                    reinterpret_cast<int64_t*>(s.a.row_ptr.data()), reinterpret_cast<int64_t*>(s.a.col_idx.data()),
                    s.a.values.data(), s.p.values.data(), s.s_diag.data());
    s.p.row_ptr = s.a.row_ptr;  // P has A's pattern (A holds no zeros)
    s.p.col_idx = s.a.col_idx;
    s.a_norm = a_norm;
    return s;
}

}  // namespace compat
}  // namespace mcmi

#endif
