// tables.cu — subsystem (1): drop filter, diagonal augmentation / splitting and
// the per-state transition tables, all on device.
//
// Reference semantics (paths relative to /root/reference/proj):
//   drop_small_entries      src/csr.cpp:127-157 (off_diagonal_range :88-105,
//                           filter_entries :109-123)
//   augment_and_split       src/split.cpp:46-100 (with_explicit_diagonal :10-42,
//                           inf_norm csr.cpp:77-86)
//   transition_probabilities src/split.cpp:102-119
//   sample_transition's CDF src/mc_engine.cpp:64-78
//
// Every per-row floating-point sum is a sequential left fold in stored order
// (one thread per row), exactly like the reference loops; maxima and minima
// are order-independent and use integer atomics on the bit patterns.  With
// -fmad=false every value here is bit-identical to the reference's.
//
// HBM layout produced (B200, 180 GB):
//   rec[n]      2 x uint4 {begin, deg, guide[16], inline forced move}
//                                            32 B per state (one sector)
//   ent[nnz_A]  double2 {cum, a/p}           16 B per transition
//   col[nnz_A]  int32                         4 B per transition
//   b1_diag[n]  f64                           8 B per state
// A step from state s reads rec[s] (1 sector), ent[begin+guide .. k] (usually
// 1 sector) and col[k]; SURVEY.md §8(d) counts 20 + 8*deg(s) algorithmic bytes
// (the full CDF row), which the guide avoids re-reading.
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {
namespace {

constexpr int TB = 256;

inline int grid_for(int64_t items, int per_block = TB) {
    int64_t g = (items + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > 148 * 8) g = 148 * 8;  // grid-stride beyond 8 blocks per SM
    return static_cast<int>(g);
}

// Block-wide reductions so each block issues ONE atomic per scalar (a per-thread
// atomic on one address serialises ~2.4M updates at L2).
__device__ __forceinline__ double block_max(double v) {
    __shared__ double red[TB / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < TB / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
    }
    __syncthreads();
    return v;  // valid in thread 0
}

__device__ __forceinline__ double block_min(double v) {
    __shared__ double red[TB / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL_MASK, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < TB / 32 ? red[threadIdx.x] : __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL_MASK, v, o));
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v) {
    __shared__ unsigned long long red[TB / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < TB / 32 ? red[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ unsigned long long block_max_u64(unsigned long long v) {
    __shared__ unsigned long long red[TB / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL_MASK, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < TB / 32 ? red[threadIdx.x] : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL_MASK, v, o));
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ double drop_threshold(const Reductions* red, double p) {
    const double mn = __longlong_as_double(static_cast<long long>(red->offmin_bits));
    const double mx = __longlong_as_double(static_cast<long long>(red->offmax_bits));
    return mn + p * (mx - mn);  // csr.cpp:136, no contraction (-fmad=false)
}

// Entry filter of drop_small_entries, evaluated in place.
struct Keep {
    int mode;           // -1 keep all, 0 value_range, 1 count_quantile (flags)
    double threshold;   // value_range
    const unsigned char* flags;
    __device__ __forceinline__ bool operator()(int64_t i, int64_t k, int64_t c, double v) const {
        if (mode < 0 || c == i) return true;  // diagonal is never dropped
        if (mode == 0) return !(fabs(v) < threshold);
        return flags[k] != 0;
    }
};

__device__ __forceinline__ Keep make_keep(const TableBuildArgs& a) {
    Keep kp;
    kp.mode = -1;
    kp.threshold = 0.0;
    kp.flags = a.keep;
    if (a.drop_fraction != 0.0) {
        if (a.drop_mode == 0) {
            // max_abs == 0 -> copy (csr.cpp:135)
            if (a.red->offmax_bits != 0ull) {
                kp.mode = 0;
                kp.threshold = drop_threshold(a.red, a.drop_fraction);
            }
        } else if (a.keep != nullptr) {
            kp.mode = 1;
        }
    }
    return kp;
}

// CSR sanity before any column is read: row_ptr[0] == 0, non-decreasing,
// row_ptr[n] == nnz.  The first offending row lands in bad_rowptr_row.
__global__ void k_validate_row_ptr(const int64_t* __restrict__ rp, int64_t n, int64_t nnz,
                                   Reductions* red) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = rp[i], b = rp[i + 1];
        if (a > b || a < 0 || b > nnz || (i == 0 && a != 0))
            atomicMin(&red->bad_rowptr_row, static_cast<long long>(i));
    }
}

// off_diagonal_range (csr.cpp:88-105).
__global__ void k_offdiag_range(TableBuildArgs a) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            if (a.col_idx[k] == i) continue;
            const double v = fabs(a.values[k]);
            mn = fmin(mn, v);
            mx = fmax(mx, v);
        }
    }
    // a thread that saw no off-diagonal contributes (+inf, 0), the identities
    mn = block_min(mn);
    mx = block_max(mx);
    if (threadIdx.x == 0 && mx >= mn) {  // block saw at least one off-diagonal
        atomic_min_nonneg(&a.red->offmin_bits, mn);
        atomic_max_nonneg(&a.red->offmax_bits, mx);
    }
}

// Pass B: ||B_reduced||inf, explicit diagonal value, column range check.
__global__ void k_rows_norm(TableBuildArgs a) {
    const Keep keep = make_keep(a);
    double best = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0, d = 0.0;
        bool found = false;
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t c = a.col_idx[k];
            const double v = a.values[k];
            if (c < 0 || c >= a.n) {
                atomicMin(&a.red->bad_col_row, static_cast<long long>(i));
                continue;
            }
            if (!keep(i, k, c, v)) continue;
            s += fabs(v);  // inf_norm: sequential row sum (csr.cpp:80-83)
            if (c == i && !found) {  // with_explicit_diagonal: missing -> 0 (split.cpp:10-42)
                d = v;
                found = true;
            }
        }
        a.diag_val[i] = d;
        best = fmax(best, s);
    }
    best = block_max(best);
    if (threadIdx.x == 0) atomic_max_nonneg(&a.red->bnorm_bits, best);
}

// Pass C: B1 = diag(B_hat), A's row counts, ||A||inf, max degree.
__global__ void k_rows_split(TableBuildArgs a) {
    const Keep keep = make_keep(a);
    const double b_norm = __longlong_as_double(static_cast<long long>(a.red->bnorm_bits));
    double best = 0.0;
    unsigned max_deg = 0;
    unsigned long long nnz_a = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = a.diag_val[i];
        double shift = a.alpha * b_norm;  // split.cpp:62-63
        if (a.mode == 1 && d < 0.0) shift = -shift;
        const double b1 = d + shift;
        a.b1_diag[i] = b1;
        if (b1 == 0.0) atomicMin(&a.red->degenerate_row, static_cast<long long>(i));
        double row_sum = 0.0;
        unsigned cnt = 0;
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t c = a.col_idx[k];
            const double v = a.values[k];
            if (c == i || c < 0 || c >= a.n || !keep(i, k, c, v)) continue;
            const double av = -v / b1;  // split.cpp:82
            if (av == 0.0) continue;
            ++cnt;
            row_sum += fabs(av);
        }
        a.a_cnt[i] = cnt;
        best = fmax(best, row_sum);
        max_deg = max(max_deg, cnt);
        nnz_a += cnt;
    }
    best = block_max(best);
    const unsigned long long md = block_max_u64(max_deg);
    nnz_a = block_sum_u64(nnz_a);
    if (threadIdx.x == 0) {
        atomic_max_nonneg(&a.red->anorm_bits, best);
        atomicMax(&a.red->max_deg, md);
        atomicAdd(&a.red->a_nnz, nnz_a);
    }
}

// Pass D: transition records (split.cpp:75-92 values, split.cpp:102-119
// probabilities, mc_engine.cpp:71-75 running CDF, mc_engine.cpp:94 ratio)
// plus the 16-bucket guide of each state's CDF.
__global__ void k_rows_fill(TableBuildArgs a) {
    const Keep keep = make_keep(a);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double b1 = a.b1_diag[i];
        const unsigned begin = a.a_off[i];
        const unsigned cnt = a.a_cnt[i];
        uint4 r0 = make_uint4(begin, cnt, 0u, 0u), r1 = make_uint4(0u, 0u, 0u, 0u);
        if (cnt > 0) {
            const int64_t k0 = a.row_ptr[i], k1 = a.row_ptr[i + 1];
            double row_sum = 0.0;  // transition_probabilities' sum == split's row_sum
            for (int64_t k = k0; k < k1; ++k) {
                const int64_t c = a.col_idx[k];
                const double v = a.values[k];
                if (c == i || c < 0 || c >= a.n || !keep(i, k, c, v)) continue;
                const double av = -v / b1;
                if (av == 0.0) continue;
                row_sum += fabs(av);
            }
            const unsigned scale = (cnt + 254u) / 255u;
            unsigned char g[kGuide];
            int m_next = 0;
            double cum = 0.0;
            unsigned o = 0;
            for (int64_t k = k0; k < k1; ++k) {
                const int64_t c = a.col_idx[k];
                const double v = a.values[k];
                if (c == i || c < 0 || c >= a.n || !keep(i, k, c, v)) continue;
                const double av = -v / b1;
                if (av == 0.0) continue;
                const double p = fabs(av) / row_sum;
                cum += p;
                const double ratio = av / p;
                if (o + 1 == cnt && cnt >= 2) cum = __longlong_as_double(0x7ff0000000000000ll);  // +inf: the fallback
                a.ent[begin + o] = make_double2(cum, ratio);
                a.col[begin + o] = static_cast<int>(c);
                if (cnt == 1) {
                    const unsigned long long rb = static_cast<unsigned long long>(__double_as_longlong(ratio));
                    r0.z = static_cast<unsigned>(rb);
                    r0.w = static_cast<unsigned>(rb >> 32);
                    r1.z = static_cast<unsigned>(c);
                }
                // guide: first o with cum_o > m/16 (m/16 exact in binary)
                while (m_next < kGuide && cum > static_cast<double>(m_next) * (1.0 / kGuide))
                    g[m_next++] = static_cast<unsigned char>(o / scale);
                ++o;
            }
            while (m_next < kGuide) g[m_next++] = static_cast<unsigned char>(cnt / scale);
            if (cnt >= 2) {
                unsigned w[4];
                for (int q = 0; q < 4; ++q)
                    w[q] = g[4 * q] | (g[4 * q + 1] << 8) | (g[4 * q + 2] << 16) |
                           (static_cast<unsigned>(g[4 * q + 3]) << 24);
                r0.z = w[0];
                r0.w = w[1];
                r1.x = w[2];
                r1.y = w[3];
                r1.w = scale;
            }
        }
        a.rec[2 * i] = r0;
        a.rec[2 * i + 1] = r1;
    }
}

// Tables straight from a caller-built SplitSystem (estimate_row on split.a /
// split.p, mc_engine.cpp:64-105): state i's transitions are P's row i in
// stored order, cum_k = sequential sum of p, ratio_k = a_k / p_k, col_k = A's
// column (P has A's pattern, test_mc_split.cpp:24-25).  No drop, no split.
__global__ void k_ap_fill(ApTableArgs a) {
    unsigned long long max_deg = 0, nnz_a = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k0 = a.row_ptr[i], k1 = a.row_ptr[i + 1];
        const unsigned begin = static_cast<unsigned>(k0);
        const unsigned cnt = static_cast<unsigned>(k1 - k0);
        uint4 r0 = make_uint4(begin, cnt, 0u, 0u), r1 = make_uint4(0u, 0u, 0u, 0u);
        const unsigned scale = (cnt + 254u) / 255u;
        unsigned char g[kGuide];
        int m_next = 0;
        double cum = 0.0;
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t c = a.col_idx[k];
            if (c < 0 || c >= a.n) atomicMin(&a.red->bad_col_row, static_cast<long long>(i));
            const double p = a.p_values[k];
            cum += p;  // sample_transition's running sum (mc_engine.cpp:71-75)
            const double ratio = a.a_values[k] / p;  // mc_engine.cpp:94
            const unsigned o = static_cast<unsigned>(k - k0);
            if (o + 1 == cnt && cnt >= 2) cum = __longlong_as_double(0x7ff0000000000000ll);  // +inf: the fallback
            a.ent[k] = make_double2(cum, ratio);
            a.col[k] = static_cast<int>(c);
            if (cnt == 1) {
                const unsigned long long rb = static_cast<unsigned long long>(__double_as_longlong(ratio));
                r0.z = static_cast<unsigned>(rb);
                r0.w = static_cast<unsigned>(rb >> 32);
                r1.z = static_cast<unsigned>(c);
            }
            while (m_next < kGuide && cum > static_cast<double>(m_next) * (1.0 / kGuide))
                g[m_next++] = static_cast<unsigned char>(o / scale);
        }
        while (m_next < kGuide) g[m_next++] = static_cast<unsigned char>(cnt / scale);
        if (cnt >= 2) {
            unsigned w[4];
            for (int q = 0; q < 4; ++q)
                w[q] = g[4 * q] | (g[4 * q + 1] << 8) | (g[4 * q + 2] << 16) |
                       (static_cast<unsigned>(g[4 * q + 3]) << 24);
            r0.z = w[0];
            r0.w = w[1];
            r1.x = w[2];
            r1.y = w[3];
            r1.w = scale;
        }
        a.rec[2 * i] = r0;
        a.rec[2 * i + 1] = r1;
        a.b1_diag[i] = 1.0;  // unused: estimate_row returns unscaled rows
        max_deg = max(max_deg, static_cast<unsigned long long>(cnt));
        nnz_a += cnt;
    }
    const unsigned long long md = block_max_u64(max_deg);
    nnz_a = block_sum_u64(nnz_a);
    if (threadIdx.x == 0) {
        atomicMax(&a.red->max_deg, md);
        atomicAdd(&a.red->a_nnz, nnz_a);
    }
}

// Rows whose L = 2 walks can use the split fold of walk.cu: r has at most
// kTriDeg transitions, each neighbour j has at most kTriNbDeg, and no neighbour
// of a neighbour is itself a neighbour of r (no triangle through r; A has no
// self loops).  Then a step-0 deposit only ever lands on a neighbour c_k with
// the fixed value ratio_k, and no step-1 deposit lands there.  O(deg^2 * deg_j)
// per row, run only for L = 2 builds.
constexpr unsigned kTriDeg = 16, kTriNbDeg = 64;
__global__ void k_tri_free(const uint4* __restrict__ rec, const int* __restrict__ col, int64_t n,
                           unsigned char* __restrict__ tri) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r0 = rec[2 * i];
        const unsigned b = r0.x, d = r0.y;
        bool tf = d >= 1 && d <= kTriDeg;
        for (unsigned a = 0; tf && a < d; ++a) {
            const uint4 q = rec[2 * static_cast<int64_t>(col[b + a])];
            if (q.y > kTriNbDeg) {
                tf = false;
                break;
            }
            for (unsigned x = 0; tf && x < q.y; ++x) {
                const int c = col[q.x + x];
                for (unsigned e = 0; e < d; ++e)
                    if (col[b + e] == c) {
                        tf = false;
                        break;
                    }
            }
        }
        tri[i] = tf ? 1 : 0;
    }
}

// ---- count-quantile drop (csr.cpp:138-155): radix select of the n_drop-th
// smallest |b_ij| over off-diagonals, ties resolved by entry position.

struct CqState {
    unsigned long long prefix, mask, target, count_less, n_drop, n_off;
    unsigned hist[256];
};

__global__ void k_cq_count(TableBuildArgs a, CqState* st) {
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) cnt += (a.col_idx[k] != i);
    cnt = block_sum_u64(cnt);
    if (threadIdx.x == 0) atomicAdd(&st->n_off, cnt);
}

__global__ void k_cq_init(CqState* st, double p) {
    // n_drop = static_cast<size_t>(p * static_cast<double>(off.size())) (csr.cpp:145-146)
    st->n_drop = static_cast<unsigned long long>(p * static_cast<double>(st->n_off));
    st->target = st->n_drop;
    st->prefix = 0;
    st->mask = 0;
    st->count_less = 0;
    for (int b = 0; b < 256; ++b) st->hist[b] = 0;
}

__global__ void k_cq_hist(TableBuildArgs a, CqState* st, int shift) {
    __shared__ unsigned h[256];
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    if (st->target != 0) {
        const unsigned long long prefix = st->prefix, mask = st->mask;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
             i += (int64_t)gridDim.x * blockDim.x)
            for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
                if (a.col_idx[k] == i) continue;
                const unsigned long long key =
                    static_cast<unsigned long long>(__double_as_longlong(fabs(a.values[k])));
                if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 255u], 1u);
            }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], h[b]);
}

__global__ void k_cq_select(CqState* st, int shift) {
    if (threadIdx.x != 0 || st->target == 0) return;
    unsigned long long before = 0;
    int b = 0;
    for (; b < 256; ++b) {
        if (before + st->hist[b] >= st->target) break;
        before += st->hist[b];
    }
    st->count_less += before;
    st->target -= before;
    st->prefix |= static_cast<unsigned long long>(b) << shift;
    st->mask |= 255ull << shift;
    for (int q = 0; q < 256; ++q) st->hist[q] = 0;
}

// tie[k] = off-diagonal entry whose |v| equals the selected threshold.
__global__ void k_cq_ties(TableBuildArgs a, const CqState* st, unsigned* tie) {
    const unsigned long long thr = st->prefix;
    const bool any = st->n_drop != 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const unsigned long long key =
                static_cast<unsigned long long>(__double_as_longlong(fabs(a.values[k])));
            tie[k] = (any && a.col_idx[k] != i && key == thr) ? 1u : 0u;
        }
}

__global__ void k_cq_keep(TableBuildArgs a, const CqState* st, const unsigned* tie_rank) {
    const unsigned long long thr = st->prefix;
    const bool any = st->n_drop != 0;
    const unsigned long long ties = st->n_drop - st->count_less;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const unsigned long long key =
                static_cast<unsigned long long>(__double_as_longlong(fabs(a.values[k])));
            bool drop = false;
            if (any && a.col_idx[k] != i)
                drop = key < thr || (key == thr && tie_rank[k] < ties);
            a.keep[k] = drop ? 0 : 1;
        }
}


// ---- the SplitSystem as matrices (mcmi_augment_and_split, §8b fine-grained
// API): the same per-row arithmetic as the table build, written out as the
// reference's b_hat / A / P CSRs (split.cpp:46-119), no drop.

// Pass 1: ||B||inf (inf_norm over all stored entries, csr.cpp:77-86), the
// first diagonal entry (with_explicit_diagonal: 0 if absent), b_hat's row
// lengths (one inserted diagonal where absent), column range.
__global__ void k_sx_norm(SplitExportArgs a) {
    double best = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0, d = 0.0;
        bool found = false;
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t c = a.col_idx[k];
            const double v = a.values[k];
            if (c < 0 || c >= a.n) atomicMin(&a.red->bad_col_row, static_cast<long long>(i));
            s += fabs(v);
            if (c == i && !found) {
                d = v;
                found = true;
            }
        }
        a.diag_val[i] = d;
        a.has_diag[i] = found ? 1 : 0;
        a.bh_cnt[i] = static_cast<int>(a.row_ptr[i + 1] - a.row_ptr[i]) + (found ? 0 : 1);
        best = fmax(best, s);
    }
    best = block_max(best);
    if (threadIdx.x == 0) atomic_max_nonneg(&a.red->bnorm_bits, best);
}

// Pass 2: b1 = d + shift, s = b1 - d (split.cpp:58-66), A's row lengths and
// ||A||inf (split.cpp:76-92).
__global__ void k_sx_split(SplitExportArgs a) {
    const double b_norm = __longlong_as_double(static_cast<long long>(a.red->bnorm_bits));
    double best = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = a.diag_val[i];
        double shift = a.alpha * b_norm;
        if (a.mode == 1 && d < 0.0) shift = -shift;
        const double b1 = d + shift;
        a.b1_diag[i] = b1;
        a.s_diag[i] = b1 - d;
        if (b1 == 0.0) atomicMin(&a.red->degenerate_row, static_cast<long long>(i));
        double row_sum = 0.0;
        int cnt = 0;
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            if (a.col_idx[k] == i) continue;
            const double av = -a.values[k] / b1;
            if (av == 0.0) continue;
            ++cnt;
            row_sum += fabs(av);
        }
        a.a_cnt[i] = cnt;
        best = fmax(best, row_sum);
    }
    best = block_max(best);
    if (threadIdx.x == 0) atomic_max_nonneg(&a.red->anorm_bits, best);
}

// Pass 3: b_hat (the first diagonal entry augmented, a missing one inserted
// before the first larger column), A and P = transition_probabilities(A)
// (split.cpp:102-119: |a| / sequential row sum; A has no zeros, so P has A's
// pattern).
__global__ void k_sx_fill(SplitExportArgs a) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double b1 = a.b1_diag[i];
        const int64_t k0 = a.row_ptr[i], k1 = a.row_ptr[i + 1];
        int64_t o = a.bh_row_ptr[i];
        bool placed = a.has_diag[i] != 0;  // with_explicit_diagonal (split.cpp:22-37)
        bool first = true;
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t c = a.col_idx[k];
            if (!placed && c > i) {
                a.bh_col[o] = i;
                a.bh_val[o++] = b1;
                placed = true;
            }
            double v = a.values[k];
            if (c == i && first) {
                v = b1;
                first = false;
            }
            a.bh_col[o] = c;
            a.bh_val[o++] = v;
        }
        if (!placed) {
            a.bh_col[o] = i;
            a.bh_val[o] = b1;
        }
        double row_sum = 0.0;
        int64_t q = a.a_row_ptr[i];
        for (int64_t k = k0; k < k1; ++k) {
            const int64_t c = a.col_idx[k];
            if (c == i) continue;
            const double av = -a.values[k] / b1;
            if (av == 0.0) continue;
            a.a_col[q] = c;
            a.a_val[q++] = av;
            row_sum += fabs(av);
        }
        for (int64_t j = a.a_row_ptr[i]; j < q; ++j) a.p_val[j] = fabs(a.a_val[j]) / row_sum;
    }
}

// transition_probabilities of an arbitrary A (split.cpp:102-119): rows with
// a zero absolute sum become empty (absorbing), the others keep A's pattern.
__global__ void k_tp_count(const int64_t* __restrict__ rp, const double* __restrict__ v, int64_t n,
                           int* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += fabs(v[k]);
        cnt[i] = s > 0.0 ? static_cast<int>(rp[i + 1] - rp[i]) : 0;
    }
}

__global__ void k_tp_fill(const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                          const double* __restrict__ v, int64_t n, const int64_t* __restrict__ out_rp,
                          int64_t* __restrict__ out_ci, double* __restrict__ out_v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (out_rp[i + 1] == out_rp[i]) continue;
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += fabs(v[k]);
        int64_t o = out_rp[i];
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            out_ci[o] = ci[k];
            out_v[o++] = fabs(v[k]) / s;
        }
    }
}

// drop_small_entries as a matrix (mcmi_drop_small_entries): the build's keep
// predicate, then filter_entries (csr.cpp:109-123) in stored order.
__global__ void k_drop_count(TableBuildArgs a, int* __restrict__ cnt) {
    const Keep keep = make_keep(a);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) c += keep(i, k, a.col_idx[k], a.values[k]) ? 1 : 0;
        cnt[i] = c;
    }
}

__global__ void k_drop_fill(TableBuildArgs a, const int64_t* __restrict__ out_rp, int64_t* __restrict__ oci,
                            double* __restrict__ ov) {
    const Keep keep = make_keep(a);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t o = out_rp[i];
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t c = a.col_idx[k];
            const double v = a.values[k];
            if (!keep(i, k, c, v)) continue;
            oci[o] = c;
            ov[o++] = v;
        }
    }
}
}  // namespace

size_t count_quantile_scratch_bytes(int64_t nnz) {
    const size_t align = 256;
    size_t b = (sizeof(CqState) + align - 1) / align * align;
    b += (static_cast<size_t>(nnz) + 1) * sizeof(unsigned) * 2 + 2 * align;  // tie, tie_rank
    b += scan_scratch_bytes(nnz) + align;
    return b;
}

cudaError_t launch_count_quantile(const TableBuildArgs& a, int64_t nnz, int64_t /*n_drop*/,
                                  void* scratch, size_t /*scratch_bytes*/, cudaStream_t s) {
    auto* base = static_cast<unsigned char*>(scratch);
    const size_t align = 256;
    CqState* st = reinterpret_cast<CqState*>(base);
    size_t off = (sizeof(CqState) + align - 1) / align * align;
    unsigned* tie = reinterpret_cast<unsigned*>(base + off);
    off += ((static_cast<size_t>(nnz) + 1) * sizeof(unsigned) + align - 1) / align * align;
    unsigned* tie_rank = reinterpret_cast<unsigned*>(base + off);
    off += ((static_cast<size_t>(nnz) + 1) * sizeof(unsigned) + align - 1) / align * align;
    void* scan_tmp = base + off;

    cudaMemsetAsync(st, 0, sizeof(CqState), s);
    const int g = grid_for(a.n);
    k_cq_count<<<g, TB, 0, s>>>(a, st);
    k_cq_init<<<1, 1, 0, s>>>(st, a.drop_fraction);
    for (int shift = 56; shift >= 0; shift -= 8) {
        k_cq_hist<<<g, TB, 0, s>>>(a, st, shift);
        k_cq_select<<<1, 32, 0, s>>>(st, shift);
    }
    k_cq_ties<<<g, TB, 0, s>>>(a, st, tie);
    cudaError_t e = scan_u32_exclusive(tie, tie_rank, nnz, scan_tmp, s);
    if (e != cudaSuccess) return e;
    k_cq_keep<<<g, TB, 0, s>>>(a, st, tie_rank);
    return cudaGetLastError();
}

cudaError_t launch_validate_row_ptr(const int64_t* row_ptr, int64_t n, int64_t nnz, Reductions* red,
                                   cudaStream_t s) {
    if (n > 0) k_validate_row_ptr<<<grid_for(n), TB, 0, s>>>(row_ptr, n, nnz, red);
    return cudaGetLastError();
}

cudaError_t launch_table_build(const TableBuildArgs& a, int64_t /*nnz*/, bool drop_active,
                               cudaStream_t s) {
    const int g = grid_for(a.n);
    if (drop_active && a.drop_mode == 0) k_offdiag_range<<<g, TB, 0, s>>>(a);
    k_rows_norm<<<g, TB, 0, s>>>(a);
    k_rows_split<<<g, TB, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_tri_free(const uint4* rec, const int* col, int64_t n, unsigned char* tri, cudaStream_t s) {
    if (n > 0) k_tri_free<<<grid_for(n), TB, 0, s>>>(rec, col, n, tri);
    return cudaGetLastError();
}

cudaError_t launch_ap_tables(const ApTableArgs& a, cudaStream_t s) {
    if (a.n > 0) k_ap_fill<<<grid_for(a.n), TB, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_table_fill(const TableBuildArgs& a, cudaStream_t s) {
    k_rows_fill<<<grid_for(a.n), TB, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_split_export(const SplitExportArgs& a, int pass, cudaStream_t s) {
    const int g = grid_for(a.n);
    if (a.n <= 0) return cudaSuccess;
    if (pass == 0) {
        k_sx_norm<<<g, TB, 0, s>>>(a);
        k_sx_split<<<g, TB, 0, s>>>(a);
    } else {
        k_sx_fill<<<g, TB, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_transition_probabilities(const int64_t* rp, const int64_t* ci, const double* v, int64_t n,
                                            int* cnt, const int64_t* out_rp, int64_t* out_ci, double* out_v,
                                            int pass, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (pass == 0) k_tp_count<<<grid_for(n), TB, 0, s>>>(rp, v, n, cnt);
    else k_tp_fill<<<grid_for(n), TB, 0, s>>>(rp, ci, v, n, out_rp, out_ci, out_v);
    return cudaGetLastError();
}

cudaError_t launch_drop_filter(const TableBuildArgs& a, bool drop_active, int pass, int* cnt, const int64_t* out_rp,
                               int64_t* oci, double* ov, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    const int g = grid_for(a.n);
    if (pass == 0) {
        if (drop_active && a.drop_mode == 0) k_offdiag_range<<<g, TB, 0, s>>>(a);
        k_drop_count<<<g, TB, 0, s>>>(a, cnt);
    } else {
        k_drop_fill<<<g, TB, 0, s>>>(a, out_rp, oci, ov);
    }
    return cudaGetLastError();
}

}  // namespace mcmi
