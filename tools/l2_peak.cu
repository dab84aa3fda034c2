// tools/l2_peak.cu — measures the B200's L2 read bandwidth (the roofline
// denominator SURVEY.md §8d asks for when the working set is L2-resident):
// 148*8 blocks stream a 48 MiB buffer (fits the 126 MB L2) 50 times with
// 128-bit loads; best of 10 launches, CUDA events.  Also a 4 GiB HBM read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/l2_peak tools/l2_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ p, size_t n, int reps, unsigned* sink) {
    unsigned acc = 0;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            const uint4 v = __ldcg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) *sink = acc;
}

static double run(size_t bytes, int reps) {
    uint4* p;
    unsigned* sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int it = 0; it < 11; ++it) {
        cudaEventRecord(a);
        rd<<<148 * 8, 512>>>(p, bytes / 16, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it > 0) best = best > bytes * (double)reps / ms / 1e6 ? best : bytes * (double)reps / ms / 1e6;
    }
    cudaFree(p);
    cudaFree(sink);
    return best;  // GB/s
}

int main() {
    const double l2 = run(size_t{48} << 20, 50);
    const double hbm = run(size_t{4} << 30, 1);
    printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"how\": \"tools/l2_peak.cu: 1184 blocks x 512 threads, 128-bit ld.global.cg; L2: 48 MiB x 50 passes, HBM: 4 GiB x 1; best of 10\"}\n", l2, hbm);
    return 0;
}
