// Host-memory probe for the drop-in's output path (C2: 159M entries, 1.28 GB
// per array).  Measures, on the GPU box's host:
//   * std::vector<int64_t>(n) value-initialisation (page faults + memset);
//   * the same after reserve + madvise(MADV_HUGEPAGE);
//   * parallel first-touch copies into fresh memory;
//   * D2H into pinned vs pageable memory; cudaHostRegister cost.
// nvcc -O2 -o /tmp/host_probe tools/host_probe.cu -lpthread
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
    const size_t n = 159458561;
    const size_t bytes = n * 8;
    std::printf("threads %u\n", std::thread::hardware_concurrency());
    for (int rep = 0; rep < 2; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<int64_t> v(n);
        std::printf("vector(n) value-init: %.1f ms\n", ms_since(t0));
    }
    for (int rep = 0; rep < 2; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<int64_t> v;
        v.reserve(n);
        uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + 4095) & ~uintptr_t(4095);
        madvise(reinterpret_cast<void*>(a), bytes - 8192, MADV_HUGEPAGE);
        v.resize(n);
        std::printf("reserve+madvise(HUGEPAGE)+resize: %.1f ms\n", ms_since(t0));
    }
#ifdef MADV_POPULATE_WRITE
    for (int T : {8, 16, 32}) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<int64_t> v;
        v.reserve(n);
        uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + 4095) & ~uintptr_t(4095);
        madvise(reinterpret_cast<void*>(a), bytes - 8192, MADV_HUGEPAGE);
        std::vector<std::thread> th;
        size_t span = (bytes - 8192) / T / 4096 * 4096;
        for (int i = 0; i < T; ++i)
            th.emplace_back([&, i] {
                size_t len = (i == T - 1) ? (bytes - 8192 - span * i) / 4096 * 4096 : span;
                madvise(reinterpret_cast<void*>(a + span * i), len, MADV_POPULATE_WRITE);
            });
        for (auto& t : th) t.join();
        double tp = ms_since(t0);
        v.resize(n);
        std::printf("T=%d reserve+hugepage+parallel POPULATE_WRITE %.1f ms, then resize total %.1f ms\n", T, tp,
                    ms_since(t0));
    }
#endif
    int64_t* src = nullptr;
    cudaMallocHost(&src, bytes);
    std::memset(src, 1, bytes);
    for (int T : {1, 8, 16, 32}) {
        auto t0 = std::chrono::steady_clock::now();
        int64_t* p = new int64_t[n];
        std::vector<std::thread> th;
        for (int i = 0; i < T; ++i)
            th.emplace_back([&, i] {
                size_t a = n * i / T, b = n * (i + 1) / T;
                std::memcpy(p + a, src + a, (b - a) * 8);
            });
        for (auto& t : th) t.join();
        double t1 = ms_since(t0);
        auto t2 = std::chrono::steady_clock::now();
        th.clear();
        for (int i = 0; i < T; ++i)
            th.emplace_back([&, i] {
                size_t a = n * i / T, b = n * (i + 1) / T;
                std::memcpy(p + a, src + a, (b - a) * 8);
            });
        for (auto& t : th) t.join();
        std::printf("T=%d pinned->fresh copy %.1f ms; pinned->touched copy %.1f ms\n", T, t1, ms_since(t2));
        delete[] p;
    }
    void* d = nullptr;
    cudaMalloc(&d, bytes);
    cudaMemset(d, 0, bytes);
    cudaDeviceSynchronize();
    for (int rep = 0; rep < 2; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        cudaMemcpy(src, d, bytes, cudaMemcpyDeviceToHost);
        std::printf("D2H pinned %.1f ms (%.1f GB/s)\n", ms_since(t0), bytes / ms_since(t0) / 1e6);
    }
    {
        std::vector<int64_t> v(n);
        for (int rep = 0; rep < 2; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            cudaMemcpy(v.data(), d, bytes, cudaMemcpyDeviceToHost);
            std::printf("D2H pageable (touched) %.1f ms\n", ms_since(t0));
        }
        auto t0 = std::chrono::steady_clock::now();
        cudaHostRegister(v.data(), bytes, cudaHostRegisterDefault);
        std::printf("cudaHostRegister %.1f ms\n", ms_since(t0));
        t0 = std::chrono::steady_clock::now();
        cudaMemcpy(v.data(), d, bytes, cudaMemcpyDeviceToHost);
        std::printf("D2H registered %.1f ms\n", ms_since(t0));
        t0 = std::chrono::steady_clock::now();
        cudaHostUnregister(v.data());
        std::printf("cudaHostUnregister %.1f ms\n", ms_since(t0));
    }
    {
        std::vector<int64_t> hv(n, 3);
        for (int rep = 0; rep < 2; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            cudaMemcpy(d, hv.data(), bytes, cudaMemcpyHostToDevice);
            std::printf("H2D pageable %.1f ms\n", ms_since(t0));
        }
        auto t0 = std::chrono::steady_clock::now();
        cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice);
        std::printf("H2D pinned %.1f ms\n", ms_since(t0));
    }
    {
        auto t0 = std::chrono::steady_clock::now();
        void* big = nullptr;
        cudaMallocHost(&big, bytes);
        std::printf("cudaMallocHost(1.28 GB) %.1f ms\n", ms_since(t0));
        cudaFreeHost(big);
    }
    return 0;
}
