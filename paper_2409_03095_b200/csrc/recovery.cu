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
// bit the same; the updates are independent across elements, so each one is a
// single bandwidth-bound pass over the n x n matrix (2 * 8 * n^2 bytes).
//
// One kernel per update.  It reads the snapshot of column/row i taken by the
// previous kernel and, for the next update j, writes the updated column j and
// row j into the other snapshot buffer, so no separate snapshot pass is needed.
// A failed update sets *err_row and every later kernel returns immediately.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

__global__ void k_snapshot(const double* __restrict__ m, int64_t n, int64_t i, double* __restrict__ col,
                           double* __restrict__ row) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        col[k] = m[k * n + i];
        row[k] = m[i * n + k];
    }
}

// Update i; snapshot of the updated column/row j (j < 0: no next update).
__global__ void k_rank1(double* __restrict__ m, int64_t n, int64_t i, double s, double tol,
                        const double* __restrict__ col, const double* __restrict__ row, int64_t j,
                        double* __restrict__ ncol, double* __restrict__ nrow, long long* err_row) {
    if (*reinterpret_cast<volatile long long*>(err_row) >= 0) return;
    const double denom = 1.0 - s * col[i];  // col[i] == M[i][i] before the update
    if (fabs(denom) <= tol) {
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *err_row = i;
        return;
    }
    const double f = s / denom;
    // blockIdx.y strides rows, threads stride columns (coalesced)
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
        const double cf = f * col[r];
        double* mr = m + r * n;
        if (cf == 0.0) {  // the reference skips the row (no -0 + 0 or inf * 0 changes)
            if (r == j)
                for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
                     c += static_cast<int64_t>(gridDim.x) * blockDim.x)
                    nrow[c] = mr[c];
            if (j >= 0 && blockIdx.x == 0 && threadIdx.x == 0) ncol[r] = mr[j];
            continue;
        }
        for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
             c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const double v = mr[c] + cf * row[c];
            mr[c] = v;
            if (r == j) nrow[c] = v;
            if (c == j) ncol[r] = v;
        }
    }
}

}  // namespace

int recover_device(double* m, int64_t n, const double* s_host, double tol, cudaStream_t st, int64_t* bad_row,
                   std::string& msg) {
    *bad_row = -1;
    if (n <= 0) return MCMI_OK;
    double *buf = nullptr;
    long long* err = nullptr;
    cudaError_t e = cudaMallocAsync(&buf, 4 * n * sizeof(double) + 16, st);
    if (e != cudaSuccess) {
        msg = std::string("alloc: ") + cudaGetErrorString(e);
        return MCMI_ENOMEM;
    }
    err = reinterpret_cast<long long*>(buf + 4 * n);
    double* snap[2][2] = {{buf, buf + n}, {buf + 2 * n, buf + 3 * n}};  // [parity][col,row]
    std::vector<int64_t> order;  // descending i with s_i != 0 (recovery.cpp:17-19)
    for (int64_t i = n; i-- > 0;)
        if (s_host[i] != 0.0) order.push_back(i);
    auto fail = [&](cudaError_t ce, const char* what) {
        msg = std::string(what) + ": " + cudaGetErrorString(ce);
        cudaFreeAsync(buf, st);
        return MCMI_ECUDA;
    };
    if ((e = cudaMemsetAsync(err, 0xff, sizeof(long long), st)) != cudaSuccess) return fail(e, "memset");
    const int threads = 256;
    const int gx = static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, 8));
    const int gy = static_cast<int>(std::min<int64_t>(n, 148 * 16 / gx));
    if (!order.empty()) {
        k_snapshot<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1184)), 256, 0, st>>>(
            m, n, order[0], snap[0][0], snap[0][1]);
        for (size_t q = 0; q < order.size(); ++q) {
            const int64_t i = order[q];
            const int64_t j = q + 1 < order.size() ? order[q + 1] : -1;
            k_rank1<<<dim3(gx, gy), threads, 0, st>>>(m, n, i, s_host[i], tol, snap[q & 1][0], snap[q & 1][1], j,
                                                       snap[(q + 1) & 1][0], snap[(q + 1) & 1][1], err);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return fail(e, "recovery kernels");
    }
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
