// Pageable -> device staging probe (the host drop-in's B upload, hostio.cpp
// stage_h2d): a host copy into pinned bounce buffers pipelined with the DMA,
// over chunk sizes, buffer counts and host threads.  Prints ms per 560 MB.
// nvcc -O2 -o tools/_build/stage_probe tools/stage_probe.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void pcopy(void* d, const void* s, size_t n, int T) {
    std::vector<std::thread> th;
    const size_t slice = ((n + T - 1) / T + 4095) / 4096 * 4096;
    for (int i = 1; i < T; ++i) {
        const size_t a = i * slice;
        if (a >= n) break;
        th.emplace_back([=] { std::memcpy(static_cast<char*>(d) + a, static_cast<const char*>(s) + a, std::min(slice, n - a)); });
    }
    std::memcpy(d, s, std::min(slice, n));
    for (auto& t : th) t.join();
}

int main() {
    const size_t bytes = size_t{560} << 20;
    std::vector<char> src(bytes, 1);
    void* dst = nullptr;
    cudaMalloc(&dst, bytes);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (size_t chunk_mb : {16, 32, 64, 128}) {
        for (int nb : {2, 3, 4}) {
            for (int T : {4, 8, 16}) {
                const size_t chunk = chunk_mb << 20;
                std::vector<void*> bb(nb);
                std::vector<cudaEvent_t> ev(nb);
                for (int i = 0; i < nb; ++i) {
                    cudaMallocHost(&bb[i], chunk);
                    cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
                }
                double best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaDeviceSynchronize();
                    const auto t0 = std::chrono::steady_clock::now();
                    std::vector<bool> used(nb, false);
                    size_t i = 0;
                    for (size_t off = 0; off < bytes; off += chunk, ++i) {
                        const int k = static_cast<int>(i % nb);
                        if (used[k]) cudaEventSynchronize(ev[k]);
                        const size_t len = std::min(chunk, bytes - off);
                        pcopy(bb[k], src.data() + off, len, T);
                        cudaMemcpyAsync(static_cast<char*>(dst) + off, bb[k], len, cudaMemcpyHostToDevice, s);
                        cudaEventRecord(ev[k], s);
                        used[k] = true;
                    }
                    cudaStreamSynchronize(s);
                    best = std::min(best, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
                }
                std::printf("chunk %3zu MB buffers %d threads %2d: %.2f ms (%.1f GB/s)\n", chunk_mb, nb, T, best,
                            bytes / best / 1e6);
                for (int i = 0; i < nb; ++i) {
                    cudaFreeHost(bb[i]);
                    cudaEventDestroy(ev[i]);
                }
            }
        }
    }
    {
        void* pin = nullptr;
        cudaMallocHost(&pin, bytes);
        std::memset(pin, 1, bytes);
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        cudaMemcpy(dst, pin, bytes, cudaMemcpyHostToDevice);
        std::printf("direct pinned H2D: %.2f ms\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        const auto t1 = std::chrono::steady_clock::now();
        pcopy(pin, src.data(), bytes, 16);
        std::printf("host copy alone (16 threads): %.2f ms\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
        const auto t2 = std::chrono::steady_clock::now();
        cudaMemcpy(dst, src.data(), bytes, cudaMemcpyHostToDevice);
        std::printf("direct pageable H2D: %.2f ms\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t2).count());
    }
    return 0;
}
