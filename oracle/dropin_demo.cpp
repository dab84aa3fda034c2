// oracle/dropin_demo.cpp — TEST INFRASTRUCTURE: the integration a reference
// maintainer would do, exercised end to end.  Uses the reference's OWN types
// and generators (/root/reference/proj/include/mcspai/*.hpp), builds M once
// with the unmodified reference (mcspai::compute_preconditioner_serial) and
// once through include/mcmi/mcspai_compat.hpp (the B200 build), and requires
// `serial.m == b200.m` (CsrMatrix::operator==, csr.hpp:39) plus equal RowMeta
// and budget.  Also swaps the Matrix Market functions and from_triplets
// (§8f rank 2) and requires identical bytes / matrices / exception types.
// `dropin_demo --io-only` runs only those (no GPU needed).
// Exit 0 = byte-identical on every case.
#include <cstdio>
#include <cstring>
#include <sstream>

#include "mcmi/mcspai_compat.hpp"
#include "mcspai/matrix_market.hpp"
#include "mcspai/mc_engine.hpp"
#include "mcspai/recovery.hpp"
#include "mcspai/dense_solve.hpp"
#include "mcspai/split.hpp"
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

static bool io_case(const char* name, const CsrMatrix& m) {
    std::ostringstream a, b;
    write_matrix_market(m, a);                      // reference
    mcmi::compat::write_matrix_market(m, b);        // B200 library
    bool ok = a.str() == b.str();
    std::istringstream in1(a.str()), in2(a.str());
    const CsrMatrix p1 = parse_matrix_market(in1);
    const CsrMatrix p2 = mcmi::compat::parse_matrix_market<CsrMatrix, ParseError>(in2);
    ok = ok && p1 == p2 && p2 == m;
    std::printf("[%s] mm %-19s n=%lld nnz=%lld bytes=%zu\n", ok ? "PASS" : "FAIL", name,
                static_cast<long long>(m.n), static_cast<long long>(m.nnz()), b.str().size());
    return ok;
}

static bool io_checks() {
    bool ok = true;
    ok &= io_case("identity8", CsrMatrix::identity(8));
    ok &= io_case("broad1024", make_broad_spectrum(1024, 24, 1e-4, 1.0, 7));
    ok &= io_case("convdiff64", make_convection_diffusion(64, 20.0, 10.0));
    // duplicates summed in the reference's sort order (3+ repeats of a coordinate)
    std::vector<index_t> r, c;
    std::vector<double> v;
    for (int k = 0; k < 5000; ++k) {
        r.push_back(k % 7);
        c.push_back((k * 31) % 5);
        v.push_back(1.0 / (k + 1) - 0.001 * (k % 13));
    }
    const CsrMatrix t1 = CsrMatrix::from_triplets(7, r, c, v);
    const CsrMatrix t2 = mcmi::compat::from_triplets<CsrMatrix>(7, r, c, v);
    std::printf("[%s] from_triplets with repeated coordinates\n", t1 == t2 ? "PASS" : "FAIL");
    ok &= t1 == t2;
    std::istringstream bad("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n");
    try {
        (void)mcmi::compat::parse_matrix_market<CsrMatrix, ParseError>(bad);
        std::printf("[FAIL] ParseError not raised\n");
        ok = false;
    } catch (const ParseError& e) {
        std::printf("[PASS] ParseError: %s\n", e.what());
    }
    return ok;
}

int main(int argc, char** argv) {
    bool ok = io_checks();
    if (argc > 1 && std::strcmp(argv[1], "--io-only") == 0) return ok ? 0 : 1;
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
    // recovery phase (§8f rank 4): recover_inverse on the reference's DenseMatrix
    {
        const CsrMatrix b = make_random_ddm(120, 0.1, 5);
        const SplitSystem sys = augment_and_split(b, 1.5, AugmentationMode::sign_aware);
        const DenseMatrix bhi = dense_inverse(csr_to_dense(sys.b_hat));
        const DenseMatrix r1 = recover_inverse(bhi, {sys.s_diag});
        const DenseMatrix r2 = mcmi::compat::recover_inverse<DenseMatrix, RecoveryError>(bhi, RecoveryPlan{sys.s_diag});
        const bool same = r1.values == r2.values;
        std::printf("[%s] recover_inverse n=%lld bit-identical\n", same ? "PASS" : "FAIL", static_cast<long long>(b.n));
        ok &= same;
    }
    // the fine-grained building blocks against the reference's own
    {
        const CsrMatrix b = make_random_ddm(300, 0.05, 11);
        bool same = true;
        for (const auto mode : {AugmentationMode::sign_aware, AugmentationMode::plain}) {
            const SplitSystem r = augment_and_split(b, 1.5, mode);
            const SplitSystem g = mcmi::compat::augment_and_split<SplitSystem, SplitError>(b, 1.5, mode);
            same &= r.b_hat == g.b_hat && r.a == g.a && r.p == g.p && r.b1_diag == g.b1_diag &&
                    r.s_diag == g.s_diag && r.a_norm == g.a_norm;
            same &= mcmi::compat::transition_probabilities(r.a) == transition_probabilities(r.a);
        }
        for (const auto dm : {DropMode::value_range, DropMode::count_quantile})
            for (const double p : {0.0, 0.2, 0.7})
                same &= mcmi::compat::drop_small_entries(b, p, dm) == drop_small_entries(b, p, dm);
        McConfig c;
        for (const double a : {0.0, 0.1, 0.5, 0.95}) {
            const ChainBudget r = derive_chain_budget(c, a);
            const ChainBudget g = mcmi::compat::derive_chain_budget<ChainBudget>(c, a);
            same &= r.n_chains == g.n_chains && r.max_len == g.max_len;
        }
        std::printf("[%s] augment_and_split / transition_probabilities / drop_small_entries / derive_chain_budget "
                    "bit-identical\n", same ? "PASS" : "FAIL");
        ok &= same;
    }
    return ok ? 0 : 1;
}
