// scatter.cu — SURVEY §8e: the multi-GPU assembly of M as one kernel over
// NVLink peer memory instead of an NCCL all-gather-v.
//
// Every rank owns a contiguous row block (distributed.partition_rows) and its
// CSR shard.  Each GPU holds one symmetric buffer (same layout on every rank,
// mapped into every peer's address space by torch's symmetric memory):
//   [row_ptr: n+1 int64][col_idx: nnz_total int64][values: nnz_total f64],
//   each array starting at a 16-byte boundary
// k_scatter_shard reads the local shard once and stores it straight into
// every peer's buffer (the local one included) at the shard's global offsets:
// row_ptr entries shifted by the shard's first entry, col/val moved as 16-byte
// vectors.  With rank order == row order this is the reference's row-ordered
// concatenation (mc_engine.cpp:214-220), so every GPU ends with the byte-
// identical M.  The stores go out over NVLink while the kernel streams the
// shard from HBM: the all-gather is the kernel's own write traffic, with no
// padding, staging or concatenation passes.  The caller orders the ranks with
// a symmetric-memory barrier afterwards.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

constexpr int kMaxPeers = 16;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t{15}; }

struct Peers {
    char* base[kMaxPeers];
    int count;
};

__global__ void k_scatter_shard(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                                const double* __restrict__ v, int64_t rows, int64_t nnz, int64_t row_off,
                                int64_t nnz_off, int64_t n_total, int64_t nnz_total, Peers p) {
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const size_t col_at = align16(static_cast<size_t>(n_total + 1) * sizeof(int64_t));
    const size_t val_at = col_at + align16(static_cast<size_t>(nnz_total) * sizeof(int64_t));
    // row pointers (rows + 1 entries; the shared boundary entry is written with
    // the same value by both neighbouring shards)
    for (int64_t r = tid; r <= rows; r += stride) {
        const int64_t x = rp[r] + nnz_off;
        for (int q = 0; q < p.count; ++q) reinterpret_cast<int64_t*>(p.base[q])[row_off + r] = x;
    }
    // entries: 16-byte vectors where the global offset keeps them aligned
    const bool vec = ((nnz_off & 1) == 0);
    if (vec) {
        const int64_t pairs = nnz / 2;
        for (int64_t k = tid; k < pairs; k += stride) {
            const longlong2 c2 = reinterpret_cast<const longlong2*>(ci)[k];
            const double2 v2 = reinterpret_cast<const double2*>(v)[k];
            for (int q = 0; q < p.count; ++q) {
                reinterpret_cast<longlong2*>(p.base[q] + col_at)[nnz_off / 2 + k] = c2;
                reinterpret_cast<double2*>(p.base[q] + val_at)[nnz_off / 2 + k] = v2;
            }
        }
        if ((nnz & 1) && tid == 0)
            for (int q = 0; q < p.count; ++q) {
                reinterpret_cast<int64_t*>(p.base[q] + col_at)[nnz_off + nnz - 1] = ci[nnz - 1];
                reinterpret_cast<double*>(p.base[q] + val_at)[nnz_off + nnz - 1] = v[nnz - 1];
            }
    } else {
        for (int64_t k = tid; k < nnz; k += stride) {
            const int64_t c = ci[k];
            const double x = v[k];
            for (int q = 0; q < p.count; ++q) {
                reinterpret_cast<int64_t*>(p.base[q] + col_at)[nnz_off + k] = c;
                reinterpret_cast<double*>(p.base[q] + val_at)[nnz_off + k] = x;
            }
        }
    }
}

}  // namespace
}  // namespace mcmi

extern "C" {

int mcmi_scatter_shard(const int64_t* row_ptr, const int64_t* col_idx, const double* values, int64_t rows,
                       int64_t nnz, int64_t row_offset, int64_t nnz_offset, int64_t n_total, int64_t nnz_total,
                       void* const* peer_buffers, int npeers, void* stream) {
    if (!row_ptr || !peer_buffers || npeers < 1 || npeers > mcmi::kMaxPeers || rows < 0 || nnz < 0 ||
        row_offset < 0 || row_offset + rows > n_total || nnz_offset < 0 || nnz_offset + nnz > nnz_total ||
        (nnz > 0 && (!col_idx || !values)))
        return MCMI_EINVAL;
    mcmi::Peers p{};
    p.count = npeers;
    for (int q = 0; q < npeers; ++q) {
        if (!peer_buffers[q]) return MCMI_EINVAL;
        p.base[q] = static_cast<char*>(peer_buffers[q]);
    }
    const int64_t work = std::max<int64_t>(rows + 1, (nnz + 1) / 2);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 8));
    mcmi::k_scatter_shard<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        row_ptr, col_idx, values, rows, nnz, row_offset, nnz_offset, n_total, nnz_total, p);
    return cudaGetLastError() == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

}  // extern "C"
