// tools/dropin_e2e.cpp — end-to-end timing of the C++ drop-in on the
// reference's own types (bench.py's "e2e_cpp" leg).
//
// A reference caller that switches to the B200 build calls
//   mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(b, cfg)
// (include/mcmi/mcspai_compat.hpp) where it called
//   mcspai::compute_preconditioner(b, cfg, n_threads)   (mc_engine.hpp:80-81;
//   callers tools/mcspai.cpp:204, bench/bench_precond.cpp:30-32)
// with B in pageable std::vectors, and receives M in std::vectors.  This
// program times exactly that call, host vectors in and out, nothing prepared
// in advance.  Only the reference's headers are used (its types); nothing of
// the reference runs.
//
//   dropin_e2e <dir with n.i64 row_ptr.i64 col_idx.i64 values.f64> eps delta alpha seed runs
// prints one JSON line: per-run ms, nnz, and a positional checksum of M
// (sum of word[i] * (2i+1) mod 2^64 over row_ptr || col_idx || value bits).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "mcmi/mcspai_compat.hpp"
#include "mcspai/mc_engine.hpp"

using namespace mcspai;

template <class T>
static std::vector<T> load(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) {
        std::fprintf(stderr, "cannot open %s\n", path.c_str());
        std::exit(2);
    }
    const std::streamsize bytes = f.tellg();
    f.seekg(0);
    std::vector<T> v(static_cast<size_t>(bytes) / sizeof(T));
    f.read(reinterpret_cast<char*>(v.data()), bytes);
    return v;
}

static uint64_t checksum(const ApproxInverse& a) {
    uint64_t s = 0, i = 0;
    auto add = [&](const void* p, size_t words) {
        const auto* w = static_cast<const uint64_t*>(p);
        for (size_t k = 0; k < words; ++k, ++i) s += w[k] * (2 * i + 1);
    };
    add(a.m.row_ptr.data(), a.m.row_ptr.size());
    add(a.m.col_idx.data(), a.m.col_idx.size());
    add(a.m.values.data(), a.m.values.size());
    return s;
}

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: dropin_e2e dir eps delta alpha seed runs\n");
        return 2;
    }
    const std::string dir = argv[1];
    CsrMatrix b;
    b.n = load<int64_t>(dir + "/n.i64").at(0);
    b.row_ptr = load<index_t>(dir + "/row_ptr.i64");
    b.col_idx = load<index_t>(dir + "/col_idx.i64");
    b.values = load<double>(dir + "/values.f64");
    McConfig cfg;
    cfg.epsilon = std::atof(argv[2]);
    cfg.delta = std::atof(argv[3]);
    cfg.alpha = std::atof(argv[4]);
    cfg.master_seed = std::strtoull(argv[5], nullptr, 10);
    const int runs = std::atoi(argv[6]);
    std::vector<double> ms;
    uint64_t sum = 0;
    long long nnz = 0;
    for (int r = 0; r <= runs; ++r) {  // run 0 is the warm-up (pinned pool, CUDA context)
        const auto t0 = std::chrono::steady_clock::now();
        ApproxInverse a = mcmi::compat::compute_preconditioner<ApproxInverse, SplitError>(b, cfg);
        const auto t1 = std::chrono::steady_clock::now();
        if (r > 0) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        if (r == runs) {
            sum = checksum(a);
            nnz = static_cast<long long>(a.m.col_idx.size());
        }
    }
    std::printf("{\"runs_ms\": [");
    for (size_t i = 0; i < ms.size(); ++i) std::printf("%s%.3f", i ? ", " : "", ms[i]);
    std::printf("], \"nnz\": %lld, \"checksum\": \"%016llx\"}\n", nnz, static_cast<unsigned long long>(sum));
    return 0;
}
