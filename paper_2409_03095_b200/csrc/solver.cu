// solver.cu — SURVEY.md §8(f) rank 1: the consumer of M on the GPU.
//
// Left-preconditioned restarted GMRES (MGS Arnoldi + Givens) and BiCGstab,
// step for step as the reference's validation solvers
// (/root/reference/proj/src/solvers.cpp:54-238): same x0 = 0, same
// preconditioned residual recurrences, same breakdown thresholds, same
// true-residual convergence contract (||rhs - B x|| / ||rhs|| <= rel_tol).
//
// Arithmetic: each SpMV row is a sequential sum in stored order and every
// axpy/scale is elementwise, so those round exactly like the reference
// (-fmad=false).  Dot products are deterministic two-level tree reductions
// (fixed launch shape), not the reference's sequential loop, so iterates drift
// at the rounding level and iteration counts agree within a small delta
// (tests/test_gpu_solver.py states it).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "mcmi.h"
#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

constexpr int ST = 256;
constexpr int kDotBlocks = 148 * 4;

struct DevCsr {
    int64_t n;
    const int64_t* rp;
    const int64_t* ci;
    const double* v;
    const int* ci32;  // int32 copy of ci (n < 2^31): half the index traffic of every SpMV
};

// y = m * x (csr.cpp:159-170): one thread per row, sequential in stored order.
__global__ void k_spmv(DevCsr m, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        const int64_t a = m.rp[i], b = m.rp[i + 1];
        if (m.ci32)
            for (int64_t k = a; k < b; ++k) s += m.v[k] * x[m.ci32[k]];
        else
            for (int64_t k = a; k < b; ++k) s += m.v[k] * x[m.ci[k]];
        y[i] = s;
    }
}

__global__ void k_cols32(const int64_t* __restrict__ ci, int64_t nnz, int* __restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = static_cast<int>(ci[k]);
}

// partial[b] = sum over the block's grid-stride slice of a[i]*b[i]
__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                              double* __restrict__ partial) {
    __shared__ double red[ST / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += a[i] * b[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < ST / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

// block b sums partial + b * nb into out[b] (b = 0 only for a single dot;
// out1 for block 1 of a paired dot)
__global__ void k_dot_final(const double* __restrict__ partial, int nb, double* __restrict__ out,
                            double* __restrict__ out1 = nullptr) {
    __shared__ double red[ST / 32];
    if (blockIdx.x == 1) {
        partial += nb;
        out = out1;
    }
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < ST / 32; ++w) t += red[w];
        *out = t;
    }
}

// k_dot_final's sum of nb partials, computed by every block of a kernel in
// the same order (so each block holds the same value); returned to all threads
__device__ __forceinline__ double block_sum_partials(const double* __restrict__ partial, int nb) {
    __shared__ double red[ST / 32];
    __shared__ double total;
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < ST / 32; ++w) t += red[w];
        total = t;
    }
    __syncthreads();
    return total;
}

// Modified Gram-Schmidt step on device (solvers.cpp:81-86): h_i = sum of the
// previous dot's partials (stored to hslot by block 0), w -= h_i * v (the
// reference's axpy with -h_i), fused with the partial sums of the next dot
// (w, u) in k_dot_partial's order (same grid, same per-thread slices), so
// every value equals the separate dot / axpy / dot sequence.
__global__ void k_mgs_step(const double* __restrict__ prev, double* __restrict__ hslot, const double* __restrict__ v,
                           double* w, const double* u, int64_t n,  // u may alias w
                           double* __restrict__ partial) {
    __shared__ double red[ST / 32];
    const double h = block_sum_partials(prev, kDotBlocks);
    if (blockIdx.x == 0 && threadIdx.x == 0) *hslot = h;
    const double a = -h;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double wi = w[i] + a * v[i];
        w[i] = wi;
        s += wi * (u == w ? wi : u[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL_MASK, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int ww = 0; ww < ST / 32; ++ww) t += red[ww];
        partial[blockIdx.x] = t;
    }
}

// h = sqrt((w, w)) from its partials (block 0 stores it), then v = w / h
// unless h < 1e-14 (the lucky-breakdown test, solvers.cpp:87-89)
__global__ void k_mgs_norm_div(const double* __restrict__ prev, double* __restrict__ hslot,
                               const double* __restrict__ w, double* __restrict__ v, int64_t n) {
    const double d = sqrt(block_sum_partials(prev, kDotBlocks));  // correctly rounded, like std::sqrt
    if (blockIdx.x == 0 && threadIdx.x == 0) *hslot = d;
    if (d < 1e-14) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = w[i] / d;
}

// y += a * x  (solvers.cpp:19-21)
__global__ void k_axpy(double a, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] += a * x[i];
}

// y = x / d
__global__ void k_div(const double* __restrict__ x, double d, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = x[i] / d;
}

// r = a - b
__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ r,
                      int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = a[i] - b[i];
}

__global__ void k_fill(double* __restrict__ y, double v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = v;
}

// ---- BiCGstab with its scalars on the device: one host round trip per
// iteration instead of five.  The scalar recurrences are the reference's
// (solvers.cpp:184-238) evaluated by every thread from device memory, so they
// round identically; the vector updates are fused but keep each element's
// sequence of operations.
struct BiState {
    double rho, alpha, omega;      // carried across iterations
    double rho1, r0v, tt, ts, rr;  // this iteration's dot products
    int flag;                      // breakdown (rho1 or r0v below 1e-30) in this iteration
    int pad;
};

// two dot products in one pass (same per-dot reduction order as k_dot_partial)
__global__ void k_dot2_partial(const double* __restrict__ a1, const double* __restrict__ b1,
                               const double* __restrict__ a2, const double* __restrict__ b2, int64_t n,
                               double* __restrict__ partial1, double* __restrict__ partial2) {
    __shared__ double red1[ST / 32], red2[ST / 32];
    double s1 = 0.0, s2 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        s1 += a1[i] * b1[i];
        s2 += a2[i] * b2[i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(FULL_MASK, s1, o);
        s2 += __shfl_xor_sync(FULL_MASK, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red1[threadIdx.x >> 5] = s1;
        red2[threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int w = 0; w < ST / 32; ++w) {
            t1 += red1[w];
            t2 += red2[w];
        }
        partial1[blockIdx.x] = t1;
        partial2[blockIdx.x] = t2;
    }
}

// p = r + beta * (p - omega * v), beta = (rho1 / rho) * (alpha / omega)   (solvers.cpp:190-199)
__global__ void k_bicg_p_dev(BiState* st, const double* __restrict__ r, const double* __restrict__ v,
                             double* __restrict__ p, int64_t n) {
    const double rho1 = st->rho1;
    if (fabs(rho1) < 1e-30) {  // breakdown: the reference stops before touching p
        if (blockIdx.x == 0 && threadIdx.x == 0) st->flag = 1;
        return;
    }
    const double beta = (rho1 / st->rho) * (st->alpha / st->omega);
    const double omega = st->omega;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = r[i] + beta * (p[i] - omega * v[i]);
}

// alpha = rho1 / r0v; s = r - alpha * v   (solvers.cpp:201-208)
__global__ void k_bicg_s_dev(BiState* st, const double* __restrict__ r, const double* __restrict__ v,
                             double* __restrict__ sv, int64_t n) {
    if (*reinterpret_cast<volatile int*>(&st->flag)) return;
    const double r0v = st->r0v;
    if (fabs(r0v) < 1e-30) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->flag = 1;
        return;
    }
    const double alpha = st->rho1 / r0v;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        sv[i] = r[i] + (-alpha) * v[i];
}

// omega = tt > 0 ? ts / tt : 0; x = (x + alpha p) + omega s; r = s - omega t   (solvers.cpp:210-220)
__global__ void k_bicg_xr_dev(BiState* st, const double* __restrict__ p, const double* __restrict__ sv,
                              const double* __restrict__ t, double* __restrict__ x, double* __restrict__ r,
                              int64_t n) {
    if (*reinterpret_cast<volatile int*>(&st->flag)) return;
    const double alpha = st->rho1 / st->r0v;
    const double tt = st->tt;
    const double omega = tt > 0.0 ? st->ts / tt : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = (x[i] + alpha * p[i]) + omega * sv[i];
        r[i] = sv[i] + (-omega) * t[i];
    }
}

// carries alpha, omega, rho to the next iteration (after every block of k_bicg_xr_dev read them)
__global__ void k_bicg_carry(BiState* st) {
    if (st->flag) return;
    const double alpha = st->rho1 / st->r0v;
    const double tt = st->tt;
    st->omega = tt > 0.0 ? st->ts / tt : 0.0;
    st->alpha = alpha;
    st->rho = st->rho1;
}

inline unsigned grid_n(int64_t n) {
    int64_t g = (n + ST - 1) / ST;
    if (g < 1) g = 1;
    if (g > 148 * 8) g = 148 * 8;
    return static_cast<unsigned>(g);
}

struct Ctx {
    cudaStream_t s;
    int64_t n;
    DevCsr b;
    DevCsr m;
    bool prec;
    double* partial;  // [kDotBlocks]
    double* scal;     // device scalar
    double* h_scal;   // pinned
    std::vector<double*> owned;
    cudaError_t err = cudaSuccess;

    double* vec() {
        double* p = nullptr;
        if (err == cudaSuccess) err = cudaMallocAsync(&p, static_cast<size_t>(n > 0 ? n : 1) * sizeof(double), s);
        if (p) owned.push_back(p);
        return p;
    }
    void spmv(const DevCsr& a, const double* x, double* y) { k_spmv<<<grid_n(n), ST, 0, s>>>(a, x, y); }
    void op(const double* x, double* y, double* tmp) {  // y = M (B x)   (solvers.cpp:23-28)
        if (prec) {
            spmv(b, x, tmp);
            spmv(m, tmp, y);
        } else {
            spmv(b, x, y);
        }
    }
    double dot(const double* a, const double* bb) {
        k_dot_partial<<<kDotBlocks, ST, 0, s>>>(a, bb, n, partial);
        k_dot_final<<<1, ST, 0, s>>>(partial, kDotBlocks, scal);
        cudaMemcpyAsync(h_scal, scal, sizeof(double), cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (err == cudaSuccess) err = e;
        return *h_scal;
    }
    double norm2(const double* a) { return std::sqrt(dot(a, a)); }
    // dot products into device slots, no host round trip
    void dot_to(const double* a, const double* bb, double* out) {
        k_dot_partial<<<kDotBlocks, ST, 0, s>>>(a, bb, n, partial);
        k_dot_final<<<1, ST, 0, s>>>(partial, kDotBlocks, out);
    }
    void dot2_to(const double* a1, const double* b1, double* out1, const double* a2, const double* b2,
                 double* out2) {
        k_dot2_partial<<<kDotBlocks, ST, 0, s>>>(a1, b1, a2, b2, n, partial, partial + kDotBlocks);
        k_dot_final<<<2, ST, 0, s>>>(partial, kDotBlocks, out1, out2);
    }
    void axpy(double a, const double* x, double* y) { k_axpy<<<grid_n(n), ST, 0, s>>>(a, x, y, n); }
    void copy(double* dst, const double* src) {
        cudaMemcpyAsync(dst, src, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToDevice, s);
    }
    double true_rel(const double* rhs, const double* x, double rhs_norm, double* tmp, double* tmp2) {
        spmv(b, x, tmp);
        k_sub<<<grid_n(n), ST, 0, s>>>(rhs, tmp, tmp2, n);
        return norm2(tmp2) / rhs_norm;
    }
    void release() {
        for (double* p : owned) cudaFreeAsync(p, s);
        owned.clear();
    }
};

// solvers.cpp:54-165
int gmres(Ctx& c, const double* rhs, double* x, const mcmi_solver_config& cfg, mcmi_solve_report& rep,
          std::string& msg) {
    const int64_t n = c.n;
    const double rhs_norm = c.norm2(rhs);
    if (rhs_norm == 0.0) {
        msg = "gmres: rhs is zero";
        return MCMI_EINVAL;
    }
    double* tmp = c.vec();
    double* tmp2 = c.vec();
    double* b_prec = c.vec();
    if (c.prec) c.spmv(c.m, rhs, b_prec);
    else c.copy(b_prec, rhs);
    const double b_prec_norm = c.norm2(b_prec);
    k_fill<<<grid_n(n), ST, 0, c.s>>>(x, 0.0, n);
    const int64_t restart = cfg.restart;
    std::vector<double*> v(static_cast<size_t>(restart + 1), nullptr);
    for (auto& p : v) p = c.vec();
    double* w = c.vec();
    double* hcol = nullptr;   // column j of H on the device
    double* h_hcol = nullptr;
    if (c.err == cudaSuccess) c.err = cudaMallocAsync(&hcol, (restart + 2) * sizeof(double), c.s);
    if (c.err == cudaSuccess) c.err = cudaMallocHost(&h_hcol, (restart + 2) * sizeof(double));
    if (c.err != cudaSuccess) return MCMI_ENOMEM;
    struct Free {
        double *d, *hh;
        cudaStream_t s;
        ~Free() {
            cudaFreeAsync(d, s);
            cudaStreamSynchronize(s);
            cudaFreeHost(hh);
        }
    } free_h{hcol, h_hcol, c.s};
    std::vector<std::vector<double>> h(restart + 1, std::vector<double>(restart, 0.0));
    std::vector<double> cs(restart), sn(restart), g(restart + 1);
    bool done = false;
    while (!done && rep.iterations < cfg.max_iters) {
        c.op(x, tmp2, tmp);
        k_sub<<<grid_n(n), ST, 0, c.s>>>(b_prec, tmp2, w, n);  // r = b_prec - M B x
        const double beta = c.norm2(w);
        if (beta < 1e-30) {
            rep.breakdown = 1;
            break;
        }
        k_div<<<grid_n(n), ST, 0, c.s>>>(w, beta, v[0], n);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int64_t j = 0;
        bool cycle_end = false;
        while (j < restart && !cycle_end) {
            c.op(v[j], w, tmp);
            // modified Gram-Schmidt with h on the device: j + 3 launches and one
            // host round trip per iteration (same dots, same axpys)
            double* pa = c.partial;
            double* pb = c.partial + kDotBlocks;
            k_dot_partial<<<kDotBlocks, ST, 0, c.s>>>(w, v[0], n, pa);
            for (int64_t i = 0; i <= j; ++i) {
                const double* u = i < j ? v[i + 1] : w;  // next dot: (w, v_{i+1}), or (w, w) for the norm
                k_mgs_step<<<kDotBlocks, ST, 0, c.s>>>(pa, hcol + i, v[i], w, u, n, pb);
                std::swap(pa, pb);
            }
            k_mgs_norm_div<<<kDotBlocks, ST, 0, c.s>>>(pa, hcol + j + 1, w, v[j + 1], n);
            cudaMemcpyAsync(h_hcol, hcol, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c.s);
            if (const cudaError_t e = cudaStreamSynchronize(c.s); e != cudaSuccess) {
                c.err = e;
                break;
            }
            for (int64_t i = 0; i <= j + 1; ++i) h[i][j] = h_hcol[i];
            const bool lucky = h[j + 1][j] < 1e-14;
            for (int64_t i = 0; i < j; ++i) {
                const double t = cs[i] * h[i][j] + sn[i] * h[i + 1][j];
                h[i + 1][j] = -sn[i] * h[i][j] + cs[i] * h[i + 1][j];
                h[i][j] = t;
            }
            const double denom = std::sqrt(h[j][j] * h[j][j] + h[j + 1][j] * h[j + 1][j]);
            if (denom < 1e-30) {
                cs[j] = 1.0;
                sn[j] = 0.0;
            } else {
                cs[j] = h[j][j] / denom;
                sn[j] = h[j + 1][j] / denom;
            }
            h[j][j] = cs[j] * h[j][j] + sn[j] * h[j + 1][j];
            h[j + 1][j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++j;
            ++rep.iterations;
            const double rel = std::abs(g[j]) / b_prec_norm;
            if (rel <= cfg.rel_tol || lucky || rep.iterations >= cfg.max_iters) {
                cycle_end = true;
                if (lucky && rel > cfg.rel_tol) rep.breakdown = 1;
            }
        }
        std::vector<double> y(static_cast<size_t>(j), 0.0);
        for (int64_t i = j; i-- > 0;) {
            double sacc = g[i];
            for (int64_t k = i + 1; k < j; ++k) sacc -= h[i][k] * y[k];
            y[i] = h[i][i] != 0.0 ? sacc / h[i][i] : 0.0;
        }
        for (int64_t k = 0; k < j; ++k) c.axpy(y[k], v[k], x);
        const double true_rel = c.true_rel(rhs, x, rhs_norm, tmp, tmp2);
        if (true_rel <= cfg.rel_tol) {
            rep.converged = 1;
            done = true;
        } else if (rep.breakdown) {
            done = true;
        }
    }
    rep.final_rel_residual = c.true_rel(rhs, x, rhs_norm, tmp, tmp2);
    rep.converged = rep.final_rel_residual <= cfg.rel_tol;
    return c.err == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

// solvers.cpp:167-238
int bicgstab(Ctx& c, const double* rhs, double* x, const mcmi_solver_config& cfg, mcmi_solve_report& rep,
             std::string& msg) {
    const int64_t n = c.n;
    const double rhs_norm = c.norm2(rhs);
    if (rhs_norm == 0.0) {
        msg = "bicgstab: rhs is zero";
        return MCMI_EINVAL;
    }
    double* tmp = c.vec();
    double* tmp2 = c.vec();
    double* b_prec = c.vec();
    double* r = c.vec();
    double* r0 = c.vec();
    double* p = c.vec();
    double* vv = c.vec();
    double* s = c.vec();
    double* t = c.vec();
    if (c.err != cudaSuccess) return MCMI_ENOMEM;
    if (c.prec) c.spmv(c.m, rhs, b_prec);
    else c.copy(b_prec, rhs);
    const double b_prec_norm = c.norm2(b_prec);
    k_fill<<<grid_n(n), ST, 0, c.s>>>(x, 0.0, n);
    c.copy(r, b_prec);
    c.copy(r0, r);
    k_fill<<<grid_n(n), ST, 0, c.s>>>(p, 0.0, n);
    k_fill<<<grid_n(n), ST, 0, c.s>>>(vv, 0.0, n);
    BiState* st = nullptr;
    BiState* h_st = nullptr;
    if (c.err == cudaSuccess) c.err = cudaMallocAsync(&st, sizeof(BiState), c.s);
    if (c.err == cudaSuccess) c.err = cudaMallocHost(&h_st, sizeof(BiState));
    if (c.err != cudaSuccess) return MCMI_ENOMEM;
    BiState init{};
    init.rho = init.alpha = init.omega = 1.0;
    *h_st = init;
    cudaMemcpyAsync(st, h_st, sizeof(BiState), cudaMemcpyHostToDevice, c.s);
    c.dot_to(r0, r, &st->rho1);
    while (rep.iterations < cfg.max_iters) {
        k_bicg_p_dev<<<grid_n(n), ST, 0, c.s>>>(st, r, vv, p, n);
        c.op(p, vv, tmp);
        c.dot_to(r0, vv, &st->r0v);
        k_bicg_s_dev<<<grid_n(n), ST, 0, c.s>>>(st, r, vv, s, n);
        c.op(s, t, tmp);
        c.dot2_to(t, t, &st->tt, t, s, &st->ts);
        k_bicg_xr_dev<<<grid_n(n), ST, 0, c.s>>>(st, p, s, t, x, r, n);
        k_bicg_carry<<<1, 1, 0, c.s>>>(st);
        // ||r||^2 for the convergence test and the next iteration's rho1 = (r0, r)
        c.dot2_to(r, r, &st->rr, r0, r, &st->rho1);
        cudaMemcpyAsync(h_st, st, sizeof(BiState), cudaMemcpyDeviceToHost, c.s);
        const cudaError_t e = cudaStreamSynchronize(c.s);
        if (e != cudaSuccess) {
            c.err = e;
            break;
        }
        if (h_st->flag) {  // rho1 or r0v breakdown: the reference stops before the update
            rep.breakdown = 1;
            break;
        }
        ++rep.iterations;
        const double rel = std::sqrt(h_st->rr) / b_prec_norm;
        if (rel <= cfg.rel_tol && c.true_rel(rhs, x, rhs_norm, tmp, tmp2) <= cfg.rel_tol) break;
        if (h_st->omega == 0.0) {
            rep.breakdown = 1;
            break;
        }
    }
    cudaFreeAsync(st, c.s);
    cudaStreamSynchronize(c.s);
    cudaFreeHost(h_st);
    rep.final_rel_residual = c.true_rel(rhs, x, rhs_norm, tmp, tmp2);
    rep.converged = rep.final_rel_residual <= cfg.rel_tol;
    return c.err == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

}  // namespace

int solve_device(const mcmi_csr_view& b, const mcmi_csr_view* m, const double* rhs_in, double* x,
                 const mcmi_solver_config& cfg, cudaStream_t s, mcmi_solve_report* rep, std::string& msg) {
    std::memset(rep, 0, sizeof(*rep));
    if (m && m->n != b.n) {
        msg = "solver: preconditioner dimension mismatch";
        return MCMI_EINVAL;
    }
    if (cfg.method == 0 && cfg.restart < 1) {
        msg = "gmres: restart must be positive";
        return MCMI_EINVAL;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    Ctx c;
    c.s = s;
    c.n = b.n;
    c.b = DevCsr{b.n, b.row_ptr, b.col_idx, b.values, nullptr};
    c.prec = m != nullptr;
    if (m) c.m = DevCsr{m->n, m->row_ptr, m->col_idx, m->values, nullptr};
    // int32 column copies for the SpMVs (one pass each, reused every iteration)
    int* ci32[2] = {nullptr, nullptr};
    if (b.n > 0 && b.n < INT32_MAX) {
        DevCsr* mats[2] = {&c.b, m ? &c.m : nullptr};
        for (int q = 0; q < 2; ++q) {
            if (!mats[q]) continue;
            int64_t nnz = 0;
            cudaMemcpyAsync(&nnz, mats[q]->rp + mats[q]->n, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (nnz > 0 && cudaMallocAsync(&ci32[q], nnz * sizeof(int), s) == cudaSuccess) {
                k_cols32<<<grid_n(nnz), ST, 0, s>>>(mats[q]->ci, nnz, ci32[q]);
                mats[q]->ci32 = ci32[q];
            }
        }
    }
    cudaMallocAsync(&c.partial, 2 * kDotBlocks * sizeof(double), s);
    cudaMallocAsync(&c.scal, sizeof(double), s);
    cudaMallocHost(&c.h_scal, sizeof(double));
    const double* rhs = rhs_in;
    double* ones_rhs = nullptr;
    if (!rhs) {  // ones_product_rhs (solvers.cpp:46-48): rhs = B * 1
        double* ones = c.vec();
        ones_rhs = c.vec();
        k_fill<<<grid_n(b.n), ST, 0, s>>>(ones, 1.0, b.n);
        c.spmv(c.b, ones, ones_rhs);
        rhs = ones_rhs;
    }
    const int code = cfg.method == 0 ? gmres(c, rhs, x, cfg, *rep, msg) : bicgstab(c, rhs, x, cfg, *rep, msg);
    c.release();
    for (int* p : ci32)
        if (p) cudaFreeAsync(p, s);
    cudaFreeAsync(c.partial, s);
    cudaFreeAsync(c.scal, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    rep->ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeHost(c.h_scal);
    if (code == MCMI_ECUDA) msg = std::string("solver: ") + cudaGetErrorString(cudaGetLastError());
    return code;
}

}  // namespace mcmi

extern "C" {

void mcmi_solver_config_default(mcmi_solver_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->method = MCMI_SOLVER_GMRES;
    c->rel_tol = 1e-6;
    c->max_iters = 30000;
    c->restart = 50;
}

int mcmi_solve_device(const mcmi_csr_view* b, const mcmi_csr_view* m, const double* rhs, double* x,
                      const mcmi_solver_config* cfg, int device, void* stream, mcmi_solve_report* rep,
                      char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    std::string msg;
    int code = MCMI_OK;
    if (!b || !x || !cfg || !rep) {
        code = MCMI_EINVAL;
        msg = "null argument";
    } else if (cudaSetDevice(device) != cudaSuccess) {
        code = MCMI_ENODEV;
        msg = "cudaSetDevice failed";
    } else {
        code = mcmi::solve_device(*b, m, rhs, x, *cfg, static_cast<cudaStream_t>(stream), rep, msg);
    }
    if (err && errlen) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return code;
}

}  // extern "C"
