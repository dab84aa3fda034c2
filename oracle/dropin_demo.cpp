// oracle/dropin_demo.cpp — TEST INFRASTRUCTURE: the integration a reference
// maintainer would do, exercised end to end.  Uses the reference's OWN types
// and generators (/root/reference/proj/include/mcspai/*.hpp), builds M once
// with the unmodified reference (mcspai::compute_preconditioner_serial) and
// once through include/mcmi/mcspai_compat.hpp (the B200 build), and requires
// `serial.m == b200.m` (CsrMatrix::operator==, csr.hpp:39) plus equal RowMeta
// and budget.  Exit 0 = byte-identical on every case.
#include <cstdio>

#include "mcmi/mcspai_compat.hpp"
#include "mcspai/mc_engine.hpp"
#include "mcspai/synthetic.hpp"

using namespace mcspai;

static bool run(const char* name, const CsrMatrix& b, const McConfig& cfg) {
    const ApproxInverse ref = compute_preconditioner_serial(b, cfg);
    const ApproxInverse gpu = mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(b, cfg);
    bool ok = ref.m == gpu.m && ref.budget_echo.n_chains == gpu.budget_echo.n_chains &&
              ref.budget_echo.max_len == gpu.budget_echo.max_len;
    for (size_t i = 0; ok && i < ref.row_meta.size(); ++i)
        ok = ref.row_meta[i].chains_used == gpu.row_meta[i].chains_used &&
             ref.row_meta[i].entries_before_retention == gpu.row_meta[i].entries_before_retention;
    std::printf("[%s] %-22s n=%lld nnz(M)=%lld\n", ok ? "PASS" : "FAIL", name,
                static_cast<long long>(b.n), static_cast<long long>(gpu.m.nnz()));
    return ok;
}

int main() {
    bool ok = true;
    McConfig defaults;
    ok &= run("poisson2d_100", make_convection_diffusion(100, 0.0, 0.0), defaults);
    McConfig acc6;  // acceptance.cpp:257-273 criterion 6 configuration
    acc6.epsilon = 0.05;
    acc6.delta = 0.01;
    acc6.alpha = 1.5;
    acc6.retain_k = 32;
    acc6.master_seed = 20260826;
    ok &= run("rdb2048_acc6", make_brusselator(32), acc6);
    McConfig bench;  // bench_precond.cpp:46-52
    bench.epsilon = 0.02;
    bench.delta = 0.01;
    bench.alpha = 1.5;
    bench.retain_k = 32;
    bench.master_seed = 42;
    ok &= run("broad1024_bench", make_broad_spectrum(1024, 24, 1e-4, 1.0, 7), bench);
    ok &= run("tridiag4096_bench", make_tridiagonal(4096), bench);
    McConfig drop = bench;
    drop.drop_fraction = 0.3;
    drop.drop_mode = DropMode::count_quantile;
    ok &= run("ddm200_quantile", make_random_ddm(200, 0.1, 3), drop);
    // error mapping: plain mode cancelling a negative diagonal (test_mc_split.cpp:89-94)
    McConfig plain;
    plain.alpha = 1.0;
    plain.mode = AugmentationMode::plain;
    const CsrMatrix two = CsrMatrix::from_triplets(2, {0, 1}, {0, 1}, {-1.0, 1.0});
    try {
        (void)mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(two, plain);
        std::printf("[FAIL] SplitError not raised\n");
        ok = false;
    } catch (const SplitError& e) {
        std::printf("[PASS] SplitError: %s\n", e.what());
    }
    return ok ? 0 : 1;
}
