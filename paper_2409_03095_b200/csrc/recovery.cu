// recovery.cu — §8f rank 4: the recovery phase (undo the diagonal
// augmentation) on the GPU, bit-identical to mcspai::recover_inverse
// (src/recovery.cpp:7-33).
//
// For i = n-1 down to 0 with s_i != 0:
//   denom = 1 - s_i * M[i][i]           (|denom| <= tol -> RecoveryError at row i)
//   f     = s_i / denom
//   M[r][c] += (f * M[r][i]) * M[i][c]  for every r with f * M[r][i] != 0
// using column i and row i as they were before update i (the reference
// snapshots them).  Every element's sequence of roundings is the reference's
// (one multiply, one multiply, one add, -fmad=false), so the result is bit for
// bit the same; the updates are independent across elements.
//
// Updates are applied in blocks of kRecK (see "blocked" below): the block's
// pivot rows, per-row coefficients and then one read-modify-write pass over M
// per kRecK updates, each element still getting exactly the reference's
// sequence of operations.  A failed update sets *err_row and every later
// kernel returns immediately.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

// ---------------------------------------------------------------- blocked
// kRecK consecutive updates u = 0..kb-1 (pivot rows/columns p_u, descending)
// in one pass over M.  With S the matrix before the block, the reference's sequence
// decomposes exactly (same operands, same order, same roundings):
//   A1  the kb x kb pivot submatrix alone evolves through the block, giving
//       f_u, CF[u][q] = f_u * S_u[p_q][p_u] (the coefficient pivot row q gets
//       at step u) and RP[u][t] = S_u[p_u][p_t] (pivot row u before step u);
//   A2  per column c, the pivot rows before their own step:
//       R_u[c] = ((S[p_u][c] + CF[0][u] R_0[c]) + CF[1][u] R_1[c]) + ...;
//   B1  per row r, its coefficients coef_u = f_u * x_u, where x_t = element
//       (r, p_t) advanced by the earlier steps: x_t += coef_u * RP[u][t];
//   B2  per element, m_rc = ((m_rc + coef_0 R_0[c]) + coef_1 R_1[c]) + ...,
//       a step skipped when its coefficient is exactly 0 (recovery.cpp:27).
// M is read and written once per K updates instead of once per update.
constexpr int kRecK = 16;
constexpr int kRecRowsPerTile = 32;

struct RecBlock {
    int64_t piv[kRecK];
    double s[kRecK];
    int kb;
};

// A1 + A2 + B1 in one launch: every block re-derives the kRecK x kRecK pivot
// evolution (A1, a few microseconds) in shared memory, then its threads take
// columns for A2 and rows for B1 (grid-stride over n for both).
__global__ void k_rec_prep(const double* __restrict__ m, int64_t n, RecBlock b, double tol,
                           double* __restrict__ R, double* __restrict__ coef, unsigned* __restrict__ nzmask,
                           long long* err_row) {
    __shared__ double S[kRecK][kRecK];
    __shared__ double CF[kRecK][kRecK];  // CF[u][q]: coefficient of pivot row q at step u
    __shared__ double RP[kRecK][kRecK];  // RP[u][t]: pivot row u before step u, at column p_t
    __shared__ double F[kRecK];
    __shared__ int bad;
    if (*reinterpret_cast<volatile long long*>(err_row) >= 0) return;
    const int kb = b.kb;
    for (int i = threadIdx.x; i < kRecK * kRecK; i += blockDim.x) {
        const int q = i / kRecK, t = i % kRecK;
        S[q][t] = (q < kb && t < kb) ? m[b.piv[q] * n + b.piv[t]] : 0.0;
    }
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int u = 0; u < kb; ++u) {
        if (threadIdx.x == 0) {
            const double denom = 1.0 - b.s[u] * S[u][u];
            if (fabs(denom) <= tol) {
                bad = 1;
                *err_row = b.piv[u];
            }
            F[u] = b.s[u] / denom;
        }
        __syncthreads();
        if (bad) return;
        double c = 0.0, r = 0.0;
        const int i = threadIdx.x;
        const int q = i / kRecK, t = i % kRecK;
        if (i < kRecK * kRecK && q < kb && t < kb) {
            c = F[u] * S[q][u];
            r = S[u][t];
        }
        __syncthreads();
        if (i < kRecK * kRecK && q < kb && t < kb) {
            if (t == 0) CF[u][q] = c;
            if (q == 0) RP[u][t] = r;
            if (c != 0.0) S[q][t] = S[q][t] + c * r;
        }
        __syncthreads();
    }
    for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < n;
         x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // A2: column x of the pivot rows before their own step
        double val[kRecK];
#pragma unroll
        for (int u = 0; u < kRecK; ++u) val[u] = u < kb ? m[b.piv[u] * n + x] : 0.0;
#pragma unroll
        for (int u = 0; u < kRecK; ++u) {
            if (u >= kb) break;
            const double ru = val[u];
            R[u * n + x] = ru;
#pragma unroll
            for (int q = u + 1; q < kRecK; ++q) {
                const double k = CF[u][q];
                if (q < kb && k != 0.0) val[q] = val[q] + k * ru;
            }
        }
        // B1: row x's coefficients
        unsigned mask = 0;
#pragma unroll
        for (int t = 0; t < kRecK; ++t) val[t] = t < kb ? m[x * n + b.piv[t]] : 0.0;
#pragma unroll
        for (int u = 0; u < kRecK; ++u) {
            if (u >= kb) break;
            const double cu = F[u] * val[u];
            coef[x * kRecK + u] = cu;
            mask |= (cu != 0.0 ? 1u : 0u) << u;
            if (cu != 0.0) {
#pragma unroll
                for (int t = u + 1; t < kRecK; ++t)
                    if (t < kb) val[t] = val[t] + cu * RP[u][t];
            }
        }
        nzmask[x] = mask;
    }
}

// B2 with RPT rows x CPT columns per thread: RPT*CPT independent chains (the
// R_u[c] registers are shared by the rows); rows whose coefficients are all
// nonzero run unrolled without per-step tests.
template <int RPT, int CPT>
__global__ void __launch_bounds__(256) k_rec_apply(double* __restrict__ m, int64_t n, int kb,
                                                    const double* __restrict__ R, const double* __restrict__ coef,
                                                    const unsigned* __restrict__ nzmask, const long long* err_row) {
    if (*reinterpret_cast<const volatile long long*>(err_row) >= 0) return;
    __shared__ __align__(16) double C[kRecRowsPerTile][kRecK];
    __shared__ unsigned MK[kRecRowsPerTile];
    int64_t col[CPT];
    double ru[CPT][kRecK];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        col[j] = (blockIdx.x * static_cast<int64_t>(CPT) + j) * blockDim.x + threadIdx.x;
#pragma unroll
        for (int u = 0; u < kRecK; ++u) ru[j][u] = (col[j] < n && u < kb) ? R[u * n + col[j]] : 0.0;
    }
    const unsigned full = kb >= 32 ? ~0u : ((1u << kb) - 1u);
    for (int64_t r0 = blockIdx.y * static_cast<int64_t>(kRecRowsPerTile); r0 < n;
         r0 += static_cast<int64_t>(gridDim.y) * kRecRowsPerTile) {
        __syncthreads();
        for (int i = threadIdx.x; i < kRecRowsPerTile * kRecK; i += blockDim.x) {
            const int64_t r = r0 + i / kRecK;
            C[i / kRecK][i % kRecK] = r < n ? coef[r * kRecK + i % kRecK] : 0.0;
        }
        for (int i = threadIdx.x; i < kRecRowsPerTile; i += blockDim.x) MK[i] = r0 + i < n ? nzmask[r0 + i] : 0u;
        __syncthreads();
        const int64_t left = n - r0;
        const int rows = left < kRecRowsPerTile ? static_cast<int>(left) : kRecRowsPerTile;
        int i = 0;
        if (kb == kRecK) {
            for (; i + RPT <= rows; i += RPT) {
                bool dense = true;
#pragma unroll
                for (int q = 0; q < RPT; ++q) dense = dense && MK[i + q] == full;
                if (!dense) break;
                double v[RPT][CPT];
#pragma unroll
                for (int q = 0; q < RPT; ++q)
#pragma unroll
                    for (int j = 0; j < CPT; ++j) v[q][j] = col[j] < n ? m[(r0 + i + q) * n + col[j]] : 0.0;
#pragma unroll
                for (int u = 0; u < kRecK; ++u) {
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const double k = C[i + q][u];
#pragma unroll
                        for (int j = 0; j < CPT; ++j) v[q][j] = v[q][j] + k * ru[j][u];
                    }
                }
#pragma unroll
                for (int q = 0; q < RPT; ++q)
#pragma unroll
                    for (int j = 0; j < CPT; ++j)
                        if (col[j] < n) m[(r0 + i + q) * n + col[j]] = v[q][j];
            }
        }
        for (; i < rows; ++i) {  // remaining rows one at a time, zero coefficients skipped
            const unsigned mk = MK[i];
            double v[CPT];
#pragma unroll
            for (int j = 0; j < CPT; ++j) v[j] = col[j] < n ? m[(r0 + i) * n + col[j]] : 0.0;
#pragma unroll
            for (int u = 0; u < kRecK; ++u) {
                if ((mk >> u) & 1u) {
                    const double k = C[i][u];
#pragma unroll
                    for (int j = 0; j < CPT; ++j) v[j] = v[j] + k * ru[j][u];
                }
            }
#pragma unroll
            for (int j = 0; j < CPT; ++j)
                if (col[j] < n) m[(r0 + i) * n + col[j]] = v[j];
        }
    }
}

}  // namespace

int recover_device(double* m, int64_t n, const double* s_host, double tol, cudaStream_t st, int64_t* bad_row,
                   std::string& msg) {
    *bad_row = -1;
    if (n <= 0) return MCMI_OK;
    std::vector<int64_t> order;  // descending i with s_i != 0 (recovery.cpp:17-19)
    for (int64_t i = n; i-- > 0;)
        if (s_host[i] != 0.0) order.push_back(i);
    // scratch: err | R[K*n] | coef[n*K] | nzmask[n]
    const size_t doubles = 2 * static_cast<size_t>(kRecK) * n + (n + 1) / 2 + 1;
    double* buf = nullptr;
    cudaError_t e = cudaMallocAsync(&buf, 16 + doubles * sizeof(double), st);
    if (e != cudaSuccess) {
        msg = std::string("alloc: ") + cudaGetErrorString(e);
        return MCMI_ENOMEM;
    }
    long long* err = reinterpret_cast<long long*>(buf);
    double* R = buf + 2;
    double* coef = R + static_cast<size_t>(kRecK) * n;
    unsigned* nzmask = reinterpret_cast<unsigned*>(coef + static_cast<size_t>(kRecK) * n);
    auto fail = [&](cudaError_t ce, const char* what) {
        msg = std::string(what) + ": " + cudaGetErrorString(ce);
        cudaFreeAsync(buf, st);
        return MCMI_ECUDA;
    };
    if ((e = cudaMemsetAsync(err, 0xff, sizeof(long long), st)) != cudaSuccess) return fail(e, "memset");
    const unsigned cols_blocks = static_cast<unsigned>((n + 255) / 256);
    const unsigned row_tiles = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>((n + kRecRowsPerTile - 1) / kRecRowsPerTile, (148 * 8 + cols_blocks - 1) / cols_blocks)));
    const unsigned lin = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 4));
    for (size_t q0 = 0; q0 < order.size(); q0 += kRecK) {
        RecBlock b{};
        b.kb = static_cast<int>(std::min<size_t>(kRecK, order.size() - q0));
        for (int u = 0; u < b.kb; ++u) {
            b.piv[u] = order[q0 + u];
            b.s[u] = s_host[order[q0 + u]];
        }
        k_rec_prep<<<lin, 256, 0, st>>>(m, n, b, tol, R, coef, nzmask, err);
        k_rec_apply<4, 2><<<dim3((cols_blocks + 1) / 2, row_tiles), 256, 0, st>>>(m, n, b.kb, R, coef, nzmask, err);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "recovery kernels");
    long long bad = -1;
    if ((e = cudaMemcpyAsync(&bad, err, sizeof bad, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return fail(e, "read status");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(e, "recovery");
    cudaFreeAsync(buf, st);
    *bad_row = bad;
    if (bad >= 0) {
        msg = "singular update at row " + std::to_string(bad);  // recovery.cpp:21-22
        return MCMI_ERECOVERY;
    }
    return MCMI_OK;
}

}  // namespace mcmi

namespace {

int finish(int code, const std::string& msg, char* err, size_t errlen) {
    if (code != MCMI_OK && err && errlen) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

// recovery.cpp:10-12: plan length, then tol
int check_args(int64_t n, const double* s_diag, int64_t s_len, double tol, std::string& msg) {
    if (n < 0 || (n > 0 && !s_diag)) {
        msg = "null argument";
        return MCMI_EINVAL;
    }
    if (s_len != n) {
        msg = "recovery plan length mismatch";
        return MCMI_EINVAL;
    }
    if (!(tol > 0.0)) {
        msg = "tol must be positive";
        return MCMI_EINVAL;
    }
    return MCMI_OK;
}

}  // namespace

extern "C" {

int mcmi_recover_inverse_device(double* m_dev, int64_t n, const double* s_diag, int64_t s_len, double tol,
                                int device, void* stream, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    std::string msg;
    int code = check_args(n, s_diag, s_len, tol, msg);
    if (code) return finish(code, msg, err, errlen);
    if (n > 0 && !m_dev) return finish(MCMI_EINVAL, "null argument", err, errlen);
    if (cudaSetDevice(device) != cudaSuccess) return finish(MCMI_ENODEV, "cudaSetDevice failed", err, errlen);
    int64_t bad = -1;
    code = mcmi::recover_device(m_dev, n, s_diag, tol, static_cast<cudaStream_t>(stream), &bad, msg);
    return finish(code, msg, err, errlen);
}

int mcmi_recover_inverse(double* m, int64_t n, const double* s_diag, int64_t s_len, double tol, int device,
                         char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    std::string msg;
    int code = check_args(n, s_diag, s_len, tol, msg);
    if (code) return finish(code, msg, err, errlen);
    if (n == 0) return MCMI_OK;
    if (!m) return finish(MCMI_EINVAL, "null argument", err, errlen);
    if (cudaSetDevice(device) != cudaSuccess) return finish(MCMI_ENODEV, "cudaSetDevice failed", err, errlen);
    cudaStream_t st = nullptr;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return finish(MCMI_ECUDA, "stream", err, errlen);
    double* d = nullptr;
    const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(n) * sizeof(double);
    cudaError_t e = cudaMallocAsync(&d, bytes, st);
    if (e != cudaSuccess) {
        cudaStreamDestroy(st);
        return finish(MCMI_ENOMEM, std::string("alloc: ") + cudaGetErrorString(e), err, errlen);
    }
    e = cudaMemcpyAsync(d, m, bytes, cudaMemcpyHostToDevice, st);
    int64_t bad = -1;
    if (e == cudaSuccess) {
        code = mcmi::recover_device(d, n, s_diag, tol, st, &bad, msg);
        if (code == MCMI_OK) {
            e = cudaMemcpyAsync(m, d, bytes, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
    }
    if (e != cudaSuccess) {
        code = MCMI_ECUDA;
        msg = std::string("recovery copies: ") + cudaGetErrorString(e);
    }
    cudaFreeAsync(d, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    return finish(code, msg, err, errlen);
}

}  // extern "C"
