// assemble.cu — device-wide exclusive scans and the CSR compaction that
// replaces the reference's serial assembly loop (mc_engine.cpp:207-225):
// row r's entries land at row_ptr[r] in row order, so the device CSR is
// byte-identical to the reference's concatenation.
#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T n = __shfl_up_sync(FULL_MASK, v, o);
        if ((threadIdx.x & 31) >= (unsigned)o) v += n;
    }
    return v;
}

template <class TI, class TA>
__global__ void k_tile_reduce(const TI* in, int64_t n, TA* partial) {
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE;
    TA s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t i = base + j * SCAN_THREADS + threadIdx.x;
        if (i < n) s += static_cast<TA>(in[i]);
    }
    s = warp_incl_scan(s);
    __shared__ TA wt[SCAN_THREADS / 32];
    if ((threadIdx.x & 31) == 31) wt[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        TA t = 0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w) t += wt[w];
        partial[blockIdx.x] = t;
    }
}

// Single block: exclusive scan of the tile partials in place; total -> *total.
template <class TA, class TO>
__global__ void k_scan_partials(TA* partial, int64_t nb, TO* total) {
    __shared__ TA carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += SCAN_THREADS) {
        const int64_t i = base + threadIdx.x;
        const TA v = i < nb ? partial[i] : TA(0);
        const TA inc = warp_incl_scan(v);
        __shared__ TA wt[SCAN_THREADS / 32];
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 31) wt[w] = inc;
        __syncthreads();
        TA wpre = 0, btot = 0;
        for (int q = 0; q < SCAN_THREADS / 32; ++q) {
            if (q < w) wpre += wt[q];
            btot += wt[q];
        }
        const TA carry = carry_s;
        if (i < nb) partial[i] = carry + wpre + inc - v;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + btot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = static_cast<TO>(carry_s);
}

template <class TI, class TA, class TO>
__global__ void k_tile_scan(const TI* in, TO* out, int64_t n, const TA* partial) {
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * (int64_t)SCAN_ITEMS;
    TA v[SCAN_ITEMS];
    TA s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t i = base + j;
        v[j] = i < n ? static_cast<TA>(in[i]) : TA(0);
        s += v[j];
    }
    const TA inc = warp_incl_scan(s);
    __shared__ TA wt[SCAN_THREADS / 32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 31) wt[w] = inc;
    __syncthreads();
    TA wpre = 0;
    for (int q = 0; q < w; ++q) wpre += wt[q];
    TA run = partial[blockIdx.x] + wpre + inc - s;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        const int64_t i = base + j;
        if (i < n) out[i] = static_cast<TO>(run);
        run += v[j];
    }
}

template <class TI, class TA, class TO>
cudaError_t scan_exclusive(const TI* in, TO* out, int64_t n, void* scratch, cudaStream_t s) {
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    TA* partial = static_cast<TA*>(scratch);
    if (nb > 0) k_tile_reduce<TI, TA><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, n, partial);
    k_scan_partials<TA, TO><<<1, SCAN_THREADS, 0, s>>>(partial, nb, out + n);
    if (nb > 0) k_tile_scan<TI, TA, TO><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, partial);
    return cudaGetLastError();
}

// Warp per row: copy the finalized row from its staging slot to the CSR,
// widening columns to the reference's int64 (csr.hpp:10).
__global__ void k_compact(const int* __restrict__ stage_col, const double* __restrict__ stage_val,
                          const int64_t* __restrict__ row_src, const int* __restrict__ row_cnt,
                          const int64_t* __restrict__ row_ptr, int64_t rows,
                          int64_t* __restrict__ col_out, double* __restrict__ val_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const int cnt = row_cnt[r];
        const int64_t src = row_src[r];
        const int64_t dst = row_ptr[r];
        for (int i = lane; i < cnt; i += 32) {
            col_out[dst + i] = stage_col[src + i];
            val_out[dst + i] = stage_val[src + i];
        }
    }
}

__global__ void k_add_offset(int64_t* __restrict__ a, int64_t add, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] += add;
}

}  // namespace

cudaError_t launch_add_offset(int64_t* a, int64_t add, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_add_offset<<<(unsigned)blocks, 256, 0, s>>>(a, add, n);
    return cudaGetLastError();
}

size_t scan_scratch_bytes(int64_t n) {
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    return static_cast<size_t>(nb + 1) * sizeof(unsigned long long);
}

cudaError_t scan_u32_exclusive(const unsigned* in, unsigned* out, int64_t n, void* scratch,
                               cudaStream_t s) {
    return scan_exclusive<unsigned, unsigned long long, unsigned>(in, out, n, scratch, s);
}

cudaError_t scan_rows_exclusive(const int* in, int64_t* out, int64_t n, void* scratch,
                                cudaStream_t s) {
    return scan_exclusive<int, long long, int64_t>(in, out, n, scratch, s);
}

cudaError_t launch_compact(const int* stage_col, const double* stage_val, const int64_t* row_src,
                           const int* row_cnt, const int64_t* row_ptr, int64_t rows,
                           int64_t* col_out, double* val_out, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    int64_t blocks = (rows * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_compact<<<(unsigned)blocks, 256, 0, s>>>(stage_col, stage_val, row_src, row_cnt, row_ptr,
                                                rows, col_out, val_out);
    return cudaGetLastError();
}

}  // namespace mcmi
