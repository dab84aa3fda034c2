// rowops.cu — the reference's per-row post-processing as batched device ops
// (SURVEY §8b fine-grained API; the build itself runs the same rules fused
// into the walk kernel's per-row finalize, walk.cu):
//
//   retain_top_k   mc_engine.cpp:124-145: keep the k entries ranked first by
//                  (column == diag_col first, |value| descending, column
//                  ascending), in the row's original order.
//   scale_columns  mc_engine.cpp:147-149: value /= b1_diag[column].
//
// Every row of a CSR is one SparseRow.  retain_top_k: one warp per row; each
// lane ranks its entries against the whole row (an entry is kept iff fewer
// than k entries precede it), then the kept entries are compacted in order
// with ballot prefix counts.  O(s^2 / 32) per row of s entries: this is the
// reference's test-level building block, not a throughput path.
#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

// (a before b) under retain_top_k's order (mc_engine.cpp:130-137); equal
// columns fall back to position so the order is total.
__device__ __forceinline__ bool topk_before(int64_t ca, double va, int64_t ia, int64_t cb, double vb, int64_t ib,
                                            int64_t diag) {
    const bool da = ca == diag, db = cb == diag;
    if (da != db) return da;
    const double ma = fabs(va), mb = fabs(vb);
    if (ma != mb) return ma > mb;
    if (ca != cb) return ca < cb;
    return ia < ib;
}

// pass 0: kept count per row; pass 1: write the kept entries at out_rp[r].
__global__ void k_topk_rows(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                            const double* __restrict__ v, int64_t n, int64_t k, const int64_t* __restrict__ diag,
                            int pass, int* __restrict__ cnt, const int64_t* __restrict__ out_rp,
                            int64_t* __restrict__ oci, double* __restrict__ ov) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const int64_t a = rp[r], s = rp[r + 1] - a;
        const bool all = k <= 0 || s <= k;  // mc_engine.cpp:125
        if (pass == 0) {
            if (lane == 0) cnt[r] = static_cast<int>(all ? s : k);
            continue;
        }
        const int64_t dcol = diag ? diag[r] : r;
        int64_t o = out_rp[r];
        for (int64_t base = 0; base < s; base += 32) {
            const int64_t i = base + lane;
            bool keep = false;
            int64_t c = 0;
            double x = 0.0;
            if (i < s) {
                c = ci[a + i];
                x = v[a + i];
                keep = all;
                if (!all) {
                    int64_t rank = 0;
                    for (int64_t j = 0; j < s && rank < k; ++j)
                        rank += topk_before(ci[a + j], v[a + j], j, c, x, i, dcol) ? 1 : 0;
                    keep = rank < k;
                }
            }
            const unsigned m = __ballot_sync(FULL_MASK, keep);
            if (keep) {
                const int64_t at = o + __popc(m & ((1u << lane) - 1u));
                oci[at] = c;
                ov[at] = x;
            }
            o += __popc(m);
        }
    }
}

__global__ void k_scale_columns(const int64_t* __restrict__ ci, const double* __restrict__ v, int64_t nnz,
                                const double* __restrict__ b1, int64_t len, double* __restrict__ out, int* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = ci[i];
        if (c < 0 || c >= len) {
            *bad = 1;
            continue;
        }
        out[i] = v[i] / b1[c];  // mc_engine.cpp:148 (-fmad=false: a plain IEEE division)
    }
}

unsigned blocks_for(int64_t items, int per_block) {
    int64_t g = (items + per_block - 1) / per_block;
    return static_cast<unsigned>(g < 1 ? 1 : g > 148 * 16 ? 148 * 16 : g);
}

}  // namespace

cudaError_t launch_topk_rows(const int64_t* rp, const int64_t* ci, const double* v, int64_t n, int64_t k,
                             const int64_t* diag, int pass, int* cnt, const int64_t* out_rp, int64_t* oci,
                             double* ov, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_topk_rows<<<blocks_for(n * 32, 256), 256, 0, s>>>(rp, ci, v, n, k, diag, pass, cnt, out_rp, oci, ov);
    return cudaGetLastError();
}

cudaError_t launch_scale_columns(const int64_t* ci, const double* v, int64_t nnz, const double* b1, int64_t b1_len,
                                 double* out, int* bad, cudaStream_t s) {
    if (nnz <= 0) return cudaSuccess;
    k_scale_columns<<<blocks_for(nnz, 256), 256, 0, s>>>(ci, v, nnz, b1, b1_len, out, bad);
    return cudaGetLastError();
}

}  // namespace mcmi
