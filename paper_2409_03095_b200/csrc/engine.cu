// engine.cu — host orchestration of the device pipeline and the C-ABI
// (include/mcmi.h).  Mirrors run_pipeline (mc_engine.cpp:153-226):
//   drop -> augment/split -> transition tables      (tables.cu, device)
//   derive_chain_budget                             (host, glibc log/ceil)
//   walk + accumulate + finalize per row            (walk.cu, device)
//   CSR assembly in row order                       (assemble.cu, device)
// There is no CPU fallback: every failure to reach the device is an error.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mcmi.h"
#include "kernels.cuh"
#include "hostio.h"

using namespace mcmi;

namespace {

struct Status {
    int code = MCMI_OK;
    std::string msg;
};

Status ok() { return {}; }
Status fail(int code, std::string msg) { return {code, std::move(msg)}; }

Status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return ok();
    cudaGetLastError();  // clear sticky non-fatal errors
    const int code = (e == cudaErrorMemoryAllocation) ? MCMI_ENOMEM
                     : (e == cudaErrorNoDevice || e == cudaErrorInvalidDevice ||
                        e == cudaErrorInsufficientDriver)
                         ? MCMI_ENODEV
                         : MCMI_ECUDA;
    return fail(code, std::string(what) + ": " + cudaGetErrorString(e));
}

#define MCMI_TRY(expr, what)                                   \
    do {                                                       \
        Status st__ = cuda_status((expr), (what));             \
        if (st__.code) return st__;                            \
    } while (0)

int report(const Status& st, char* err, size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, st.msg.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return st.code;
}

// Grow-only device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes == 0) bytes = 1;
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = bytes + bytes / 8;
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) return e;
        cap = want;
        return cudaSuccess;
    }
    // Grow keeping the first `keep` bytes (stream-ordered copy).
    cudaError_t grow_preserve(size_t bytes, size_t keep, cudaStream_t s) {
        if (bytes <= cap) return cudaSuccess;
        void* q = nullptr;
        const size_t want = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&q, want);
        if (e != cudaSuccess) return e;
        if (p && keep) {
            e = cudaMemcpyAsync(q, p, keep, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return e;
        }
        if (p) cudaFree(p);
        p = q;
        cap = want;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int64_t next_pow2(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

int64_t sat_mul(int64_t a, int64_t b) {
    if (a <= 0 || b <= 0) return 0;
    if (a > INT64_MAX / b) return INT64_MAX;
    return a * b;
}

// derive_chain_budget (mc_engine.cpp:12-33), on the host so glibc's log and
// ceil give the reference's exact (N, L).
// static_cast<index_t>(double) as the reference's x86-64 build executes it
// (cvttsd2si): out-of-range and NaN inputs give INT64_MIN.  The cast is UB in
// C++, but this is what the reference binary computes (e.g. ||A|| -> 1 makes
// N = max(1, INT64_MIN) = 1), so the drop-in reproduces it.
int64_t x86_cvt(double x) {
    return (x >= -9223372036854775808.0 && x < 9223372036854775808.0) ? static_cast<int64_t>(x) : INT64_MIN;
}

Status chain_budget(const mcmi_config& c, double a_norm, int64_t* nc, int64_t* ml) {
    if (!(a_norm >= 0.0 && a_norm < 1.0)) return fail(MCMI_EINVAL, "||A|| must lie in [0,1)");
    int64_t n_chains, max_len;
    if (c.has_chains_override) {
        n_chains = c.chains_override;
    } else {
        const double root = 0.6745 / (c.epsilon * (1.0 - a_norm));
        n_chains = x86_cvt(std::ceil(root * root));
    }
    if (c.has_max_len_override) {
        max_len = c.max_len_override;
    } else if (a_norm <= 0.0) {
        max_len = 1;
    } else {
        const double len = std::log(c.delta) / std::log(a_norm);
        max_len = std::max<int64_t>(1, x86_cvt(std::ceil(len)));
    }
    n_chains = std::max<int64_t>(1, n_chains);
    *nc = n_chains;
    *ml = max_len;
    return ok();
}

}  // namespace

// ---------------------------------------------------------------- engine

struct mcmi_engine {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own = nullptr;
    cudaEvent_t ev[6] = {};
    DevBuf red, diag_val, a_cnt, a_off, keep, rec, ent, colA, b1, scan_tmp, cq_tmp;
    DevBuf stage_col, stage_val, row_cnt, row_src, chains_used, entries_before, counters;
    DevBuf ovf[2];
    DevBuf tri;  // L = 2 split-fold row flags
    DevBuf gscratch;  // global accumulator tier
    DevBuf out_rp, out_col, out_val;
    // streamed build (mcmi_build_into): double-buffered output slabs + copy stream
    DevBuf col_slab[2], val_slab[2];
    cudaStream_t copy = nullptr;
    cudaEvent_t copy_done[2] = {};
    cudaEvent_t chunk_ready = nullptr;
    cudaError_t ensure_copy_stream() {
        if (copy) return cudaSuccess;
        cudaError_t r = cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking);
        for (auto& ev : copy_done)
            if (r == cudaSuccess) r = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (r == cudaSuccess) r = cudaEventCreateWithFlags(&chunk_ready, cudaEventDisableTiming);
        if (r == cudaSuccess)  // both slabs start released
            for (auto& ev : copy_done) cudaEventRecord(ev, copy);
        return r;
    }
    Reductions* h_red = nullptr;          // pinned
    unsigned long long* h_ctr = nullptr;  // pinned [8]
    int64_t* h_i64 = nullptr;             // pinned [4]
    int64_t* h_pilot = nullptr;           // pinned pilot-row RowMeta
    size_t h_pilot_n = 0;
    int64_t* h_pilot_buf(size_t count) {
        if (count > h_pilot_n) {
            if (h_pilot) cudaFreeHost(h_pilot);
            h_pilot = nullptr;
            h_pilot_n = 0;
            if (cudaMallocHost(&h_pilot, count * sizeof(int64_t)) != cudaSuccess) return nullptr;
            h_pilot_n = count;
        }
        return h_pilot;
    }
};

namespace {

Status engine_init(mcmi_engine* e, int device) {
    int count = 0;
    MCMI_TRY(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count)
        return fail(MCMI_ENODEV, "CUDA device " + std::to_string(device) + " not present (" +
                                     std::to_string(count) + " visible)");
    e->device = device;
    MCMI_TRY(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    MCMI_TRY(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major < 10)
        return fail(MCMI_ENODEV, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
    e->num_sms = prop.multiProcessorCount;
    MCMI_TRY(cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& ev : e->ev) MCMI_TRY(cudaEventCreate(&ev), "cudaEventCreate");
    MCMI_TRY(cudaMallocHost(&e->h_red, sizeof(Reductions)), "cudaMallocHost");
    MCMI_TRY(cudaMallocHost(&e->h_ctr, 8 * sizeof(unsigned long long)), "cudaMallocHost");
    MCMI_TRY(cudaMallocHost(&e->h_i64, 4 * sizeof(int64_t)), "cudaMallocHost");
    // keep stream-ordered allocations (host-API input staging) cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return ok();
}

void engine_release(mcmi_engine* e) {
    cudaSetDevice(e->device);
    for (DevBuf* b : {&e->red, &e->diag_val, &e->a_cnt, &e->a_off, &e->keep, &e->rec, &e->ent,
                      &e->colA, &e->b1, &e->scan_tmp, &e->cq_tmp, &e->stage_col, &e->stage_val,
                      &e->row_cnt, &e->row_src, &e->chains_used, &e->entries_before,
                      &e->counters, &e->ovf[0], &e->ovf[1], &e->tri, &e->gscratch, &e->out_rp, &e->out_col,
                      &e->out_val, &e->col_slab[0], &e->col_slab[1],
                      &e->val_slab[0], &e->val_slab[1]})
        b->release();
    for (auto& ev : e->copy_done)
        if (ev) cudaEventDestroy(ev);
    if (e->chunk_ready) cudaEventDestroy(e->chunk_ready);
    if (e->copy) cudaStreamDestroy(e->copy);
    for (auto& ev : e->ev)
        if (ev) cudaEventDestroy(ev);
    if (e->own) cudaStreamDestroy(e->own);
    if (e->h_red) cudaFreeHost(e->h_red);
    if (e->h_ctr) cudaFreeHost(e->h_ctr);
    if (e->h_i64) cudaFreeHost(e->h_i64);
    if (e->h_pilot) cudaFreeHost(e->h_pilot);
}

constexpr int kLogMax = 256;         // deposit-log entries per warp (shared memory)
constexpr int64_t kMaxWalkLen = 1 << 16;  // longest walk (log capacity of the global tier)
constexpr int64_t kMaxSmemWalkLen = 256;  // longer max_len go straight to the global tier
constexpr int64_t kLongRowDeposits = 1 << 15;  // N * L from which the pilot sizes by waves

struct Tier {
    int cap, cap_limit, lanes, log_stride, warps_per_block;
    bool global = false;  // accumulator + log in global scratch
};

Tier make_tier(int cap, int64_t max_len) {
    Tier t;
    t.cap = cap;
    t.cap_limit = cap - cap / 4;
    const int64_t s64 = std::max<int64_t>(1, max_len);
    t.log_stride = static_cast<int>(std::min<int64_t>(s64, INT_MAX / 64));
    const int logmax = std::max(kLogMax, t.log_stride);
    t.lanes = std::max(1, std::min(32, logmax / t.log_stride));
    const size_t per_warp = walk_smem_bytes_per_warp(t.cap, t.lanes, t.log_stride);
    t.warps_per_block = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, (96u * 1024u) / per_warp)));
    return t;
}

// Global-memory tier: any row size, full-width batches for long walks.
Tier make_global_tier(int64_t bound, int64_t max_len, int64_t min_cap = 8192) {
    Tier t;
    int64_t cap = min_cap;
    while (cap - cap / 4 < bound && cap < (int64_t{1} << 30)) cap <<= 1;
    t.cap = static_cast<int>(cap);
    t.cap_limit = t.cap - t.cap / 4;
    t.log_stride = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, max_len), kMaxWalkLen));
    t.lanes = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(32, (int64_t{1} << 16) / t.log_stride)));
    t.warps_per_block = 8;
    t.global = true;
    return t;
}

// Host destination of a streamed build (mcmi_build_into: caller-owned arrays;
// mcmi_build / mcmi_job_*: library-owned pinned buffers that grow on demand).
struct HostSink {
    int64_t* row_ptr = nullptr;  // [rows + 1]
    int64_t* col_idx = nullptr;
    double* values = nullptr;
    int64_t capacity = 0;  // entries col_idx / values hold
    int64_t* chains_used = nullptr;
    int64_t* entries_before = nullptr;
    // Library-owned output: called (copy stream drained) when entries [0, need)
    // must fit; may re-point col_idx / values keeping entries [0, have).
    // `estimate` extrapolates the final entry count from the rows built so far.
    std::function<Status(HostSink&, int64_t need, int64_t estimate, int64_t have)> grow;
    // After each row chunk's entry count is known: (rows done, entries so far, rows).
    std::function<void(int64_t, int64_t, int64_t)> progress;
    // After a chunk's entries [lo, hi) are queued for copy on stream `copy`.
    std::function<void(int64_t lo, int64_t hi, cudaStream_t copy)> queued;
    double first_chunk = 0.0;  // > 0: fraction of the rows in the first chunk (an early estimate)
};

// Device staging budget of one row chunk (stage_col + stage_val); rows are
// walked in chunks when rows x slot stride would exceed it.
int64_t staging_budget_bytes() {
    const char* v = getenv("MCMI_STAGE_BUDGET_MB");  // tests / tuning
    return v && *v ? std::max<int64_t>(1, atoll(v)) << 20 : int64_t{8} << 30;
}

// estimate_row on a caller-built SplitSystem (mcmi_estimate_rows): `b` is then
// split.a, the tables come from A and P's values, the budget is the caller's.
struct ApSource {
    const double* p_values;  // device, on A's pattern
    int64_t n_chains, max_len;
};

Status engine_build(mcmi_engine* e, const mcmi_csr_view& b, const mcmi_config& cfg,
                    int64_t row_begin, int64_t row_end, cudaStream_t s, mcmi_device_csr* out,
                    mcmi_stats* stats, HostSink* sink = nullptr, const ApSource* ap = nullptr) {
    const int64_t n = b.n;
    mcmi_stats st{};
    if (n < 0) return fail(MCMI_EINVAL, "negative dimension");
    if (n > INT_MAX - 1) return fail(MCMI_EINVAL, "dimension exceeds 2^31-2 rows");
    if (row_begin < 0) row_begin = 0;
    if (row_end < 0 || row_end > n) row_end = n;
    if (row_end < row_begin) row_end = row_begin;
    const int64_t rows = row_end - row_begin;
    // csr.cpp:128-129 comes first in the reference pipeline, then split.cpp:48
    if (!(cfg.drop_fraction >= 0.0 && cfg.drop_fraction <= 1.0))
        return fail(MCMI_EINVAL, "drop fraction must lie in [0,1]");
    if (!(cfg.alpha > 0.0)) return fail(MCMI_EINVAL, "alpha must be positive");
    if (cfg.rng_mode != MCMI_RNG_REFERENCE && cfg.rng_mode != MCMI_RNG_KEYED)
        return fail(MCMI_EINVAL, "rng_mode must be MCMI_RNG_REFERENCE or MCMI_RNG_KEYED");
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");

    MCMI_TRY(cudaEventRecord(e->ev[0], s), "cudaEventRecord");
    int64_t nnz = 0;
    if (n > 0) {
        MCMI_TRY(cudaMemcpyAsync(e->h_i64, b.row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                 "read row_ptr[n]");
        MCMI_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        nnz = e->h_i64[0];
        if (nnz < 0) return fail(MCMI_EINVAL, "row_ptr[n] is negative");
    }
    const int64_t n1 = std::max<int64_t>(n, 1);
    const int64_t z1 = std::max<int64_t>(nnz, 1);

    // ---- subsystem 1: tables
    MCMI_TRY(e->red.ensure(sizeof(Reductions)), "alloc");
    MCMI_TRY(e->diag_val.ensure(n1 * sizeof(double)), "alloc diag");
    MCMI_TRY(e->a_cnt.ensure(n1 * sizeof(unsigned)), "alloc a_cnt");
    MCMI_TRY(e->a_off.ensure((n1 + 1) * sizeof(unsigned)), "alloc a_off");
    MCMI_TRY(e->rec.ensure(2 * n1 * sizeof(uint4)), "alloc rec");
    MCMI_TRY(e->ent.ensure((z1 + 2) * sizeof(double2)), "alloc ent");  // +2: aligned pair loads
    MCMI_TRY(e->colA.ensure((z1 + 2) * sizeof(int)), "alloc col");
    MCMI_TRY(e->b1.ensure(n1 * sizeof(double)), "alloc b1");
    MCMI_TRY(e->scan_tmp.ensure(scan_scratch_bytes(std::max(n1, z1)) + 64), "alloc scan");

    Reductions init{};
    init.offmin_bits = 0x7ff0000000000000ull;
    init.degenerate_row = LLONG_MAX;
    init.bad_col_row = LLONG_MAX;
    init.bad_rowptr_row = LLONG_MAX;
    *e->h_red = init;
    MCMI_TRY(cudaMemcpyAsync(e->red.p, e->h_red, sizeof(Reductions), cudaMemcpyHostToDevice, s),
             "init reductions");

    // row_ptr must be a valid CSR row pointer before any column is read
    if (n > 0) {
        MCMI_TRY(launch_validate_row_ptr(b.row_ptr, n, nnz, e->red.as<Reductions>(), s), "validate row_ptr");
        MCMI_TRY(cudaMemcpyAsync(e->h_red, e->red.p, sizeof(Reductions), cudaMemcpyDeviceToHost, s),
                 "read validation");
        MCMI_TRY(cudaStreamSynchronize(s), "validate row_ptr");
        if (e->h_red->bad_rowptr_row != LLONG_MAX)
            return fail(MCMI_EINVAL, "row_ptr is not a valid CSR row pointer at row " +
                                         std::to_string(e->h_red->bad_rowptr_row));
        st.launches += 1;
    }

    TableBuildArgs ta{};
    ta.n = n;
    ta.row_ptr = b.row_ptr;
    ta.col_idx = b.col_idx;
    ta.values = b.values;
    ta.drop_fraction = cfg.drop_fraction;
    ta.drop_mode = cfg.drop_mode;
    ta.alpha = cfg.alpha;
    ta.mode = cfg.mode == MCMI_AUGMENT_PLAIN ? 0 : 1;
    ta.red = e->red.as<Reductions>();
    ta.diag_val = e->diag_val.as<double>();
    ta.a_cnt = e->a_cnt.as<unsigned>();
    ta.a_off = e->a_off.as<unsigned>();
    ta.keep = nullptr;
    ta.rec = e->rec.as<uint4>();
    ta.ent = e->ent.as<double2>();
    ta.col = e->colA.as<int>();
    ta.b1_diag = e->b1.as<double>();
    const bool drop_active = !ap && cfg.drop_fraction != 0.0 && n > 0;
    const int64_t scan_launches_n = (n > 0 ? 3 : 1);
    if (ap) {
        if (nnz >= (int64_t{1} << 32)) return fail(MCMI_EINVAL, "A has 2^32 or more entries");
        const ApTableArgs aa{n,          b.row_ptr,  b.col_idx, b.values, ap->p_values, e->red.as<Reductions>(),
                             ta.rec,     ta.ent,     ta.col,    ta.b1_diag};
        MCMI_TRY(launch_ap_tables(aa, s), "tables from A and P");
        st.launches += n > 0 ? 1 : 0;
    } else if (drop_active && cfg.drop_mode == MCMI_DROP_COUNT_QUANTILE) {
        MCMI_TRY(e->keep.ensure(z1), "alloc keep");
        MCMI_TRY(e->cq_tmp.ensure(count_quantile_scratch_bytes(z1)), "alloc cq");
        ta.keep = e->keep.as<unsigned char>();
        MCMI_TRY(launch_count_quantile(ta, nnz, 0, e->cq_tmp.p, e->cq_tmp.cap, s), "count-quantile drop");
        st.launches += 2 + 2 * 8 + 1 + (nnz > 0 ? 3 : 1) + 1;
    }
    if (n > 0 && !ap) {
        MCMI_TRY(launch_table_build(ta, nnz, drop_active, s), "table build");
        MCMI_TRY(scan_u32_exclusive(ta.a_cnt, ta.a_off, n, e->scan_tmp.p, s), "scan a_cnt");
        MCMI_TRY(launch_table_fill(ta, s), "table fill");
        st.launches += (drop_active && cfg.drop_mode == MCMI_DROP_VALUE_RANGE ? 3 : 2) + scan_launches_n + 1;
    }
    MCMI_TRY(cudaMemcpyAsync(e->h_red, e->red.p, sizeof(Reductions), cudaMemcpyDeviceToHost, s),
             "read reductions");
    MCMI_TRY(cudaEventRecord(e->ev[1], s), "cudaEventRecord");
    MCMI_TRY(cudaStreamSynchronize(s), "table build");
    const Reductions red = *e->h_red;
    if (red.bad_col_row != LLONG_MAX)
        return fail(MCMI_ERANGE, "column index out of range in row " + std::to_string(red.bad_col_row));
    double a_norm = 0.0;
    int64_t N = 1, L = 1;
    if (ap) {
        N = ap->n_chains;
        L = ap->max_len;
        if (N < 1) return fail(MCMI_EINVAL, "n_chains must be positive");
    } else {
        if (red.degenerate_row != LLONG_MAX)  // split.cpp:67-69
            return fail(MCMI_ESPLIT, "degenerate diagonal after augmentation at row " +
                                         std::to_string(red.degenerate_row));
        std::memcpy(&a_norm, &red.anorm_bits, sizeof(double));
        if (!(a_norm < 1.0))  // split.cpp:94-96
            return fail(MCMI_ESPLIT, "diagonal dominance failure: ||A||inf = " + std::to_string(a_norm));
        if (red.a_nnz >= (1ull << 32)) return fail(MCMI_EINVAL, "A has 2^32 or more entries");
        Status bs = chain_budget(cfg, a_norm, &N, &L);
        if (bs.code) return bs;
    }
    if (N > INT_MAX) return fail(MCMI_EINVAL, "chain budget exceeds 2^31-1 chains per row");
    // walk lengths: the deposit log holds min(L, 65536) steps per chain; a walk
    // that would outgrow its tier's log overflows the row to the next tier, and
    // only walks actually longer than 65536 steps are refused
    st.n_chains = N;
    st.max_len = L;
    st.a_norm = a_norm;
    st.rows = rows;

    // ---- subsystems 2 + 3: walks, accumulate, finalize
    const int64_t dmax = static_cast<int64_t>(red.max_deg);
    int64_t reach = 1, term = 1;  // 1 + d + d^2 + ... + d^L (saturating)
    for (int64_t t = 0; t < std::max<int64_t>(L, 0) && reach < (1 << 20); ++t) {
        term = sat_mul(term, dmax);
        if (term == 0) break;
        reach = (reach > INT64_MAX - term) ? INT64_MAX : reach + term;
    }
    const int64_t deposits = sat_mul(N, std::max<int64_t>(L, 0));  // distinct <= 1 + N*L
    int64_t bound = std::min<int64_t>(n1, reach);
    if (deposits < INT64_MAX) bound = std::min<int64_t>(bound, deposits + 1);
    // Tiers: shared-memory tables up to 256 slots (48 warps/SM), then a 1024-slot
    // tier and the tier sized to the bound, both in global scratch (32 warps/SM).
    // A 1024-slot table in shared memory fits 16 warps/SM, too few to cover the
    // DRAM latency of the walks that need it (C5: 1.25x slower, profiles/
    // r01_c5_l8_walk_summary.txt); from global scratch it is L2-resident.
    int first_cap = static_cast<int>(std::min<int64_t>(256, std::max<int64_t>(32, next_pow2((bound * 4 + 2) / 3))));
    std::vector<Tier> tiers;
    if (L <= kMaxSmemWalkLen) {
        tiers.push_back(make_tier(first_cap, L));
        if (first_cap < 256 && tiers.back().cap_limit < bound) tiers.push_back(make_tier(256, L));
        if (tiers.back().cap_limit < bound) tiers.push_back(make_global_tier(0, L, 1024));
    }
    // Global tiers grow x8 up to the one sized to the bound: a row lands in a
    // table within 8x of its distinct columns, so huge bounds (C5's 10^4 x 32
    // corner: bound 3.2e5, rows of far fewer columns) do not give every warp
    // a multi-MB table (fewer resident warps, a finalize scan of cap slots).
    {
        int64_t gcap = (!tiers.empty() && tiers.back().global) ? int64_t{tiers.back().cap} * 8 : 8192;
        while (tiers.empty() || tiers.back().cap_limit < bound) {
            const Tier t = make_global_tier(0, L, gcap);
            if (t.cap_limit >= bound || gcap >= (int64_t{1} << 27)) {
                tiers.push_back(make_global_tier(bound, L));  // the smallest table holding the bound
                break;
            }
            tiers.push_back(t);
            gcap *= 8;
        }
    }
    st.hash_cap = first_cap;  // updated below if the pilot starts on a larger tier

    MCMI_TRY(e->row_cnt.ensure(std::max<int64_t>(rows, 1) * sizeof(int)), "alloc row_cnt");
    MCMI_TRY(e->row_src.ensure(std::max<int64_t>(rows, 1) * sizeof(int64_t)), "alloc row_src");
    MCMI_TRY(e->chains_used.ensure(std::max<int64_t>(rows, 1) * sizeof(int64_t)), "alloc meta");
    MCMI_TRY(e->entries_before.ensure(std::max<int64_t>(rows, 1) * sizeof(int64_t)), "alloc meta");
    MCMI_TRY(e->counters.ensure(8 * sizeof(unsigned long long)), "alloc counters");
    MCMI_TRY(e->ovf[0].ensure(std::max<int64_t>(rows, 1) * sizeof(int)), "alloc overflow");
    MCMI_TRY(e->ovf[1].ensure(std::max<int64_t>(rows, 1) * sizeof(int)), "alloc overflow");

    auto stride_of = [&](const Tier& t) -> int64_t {
        int64_t sst = std::min<int64_t>(t.cap_limit, bound);
        if (cfg.retain_k > 0) sst = std::min<int64_t>(sst, cfg.retain_k);
        return std::max<int64_t>(sst, 1);
    };
    // L = 2: flag the rows whose walks can use the split fold (walk.cu); the
    // test is O(deg^2 deg_j) per row, so only for matrices of small degree
    const unsigned char* tri = nullptr;
    if (L == 2 && n > 0 && dmax <= 16 && !getenv("MCMI_WALK_NO_SPLIT")) {
        MCMI_TRY(e->tri.ensure(n1), "alloc tri");
        MCMI_TRY(launch_tri_free(e->rec.as<uint4>(), e->colA.as<int>(), n, e->tri.as<unsigned char>(), s), "tri");
        st.launches += 1;
        tri = e->tri.as<unsigned char>();
    }
    // Resident warps of a global-scratch tier: one table per warp, up to 32
    // warps/SM.  Global-tier tables are latency-bound (random probes into HBM),
    // so resident warps are throughput: up to half of the free memory, 64 GB
    // (MCMI_SCRATCH_GB), is scratch.
    auto global_warps = [&](const Tier& t, int64_t* warps) -> Status {
        const size_t per_warp = walk_global_bytes_per_warp(t.cap, t.lanes, t.log_stride);
        const int64_t full = static_cast<int64_t>(e->num_sms) * kGlWarpsPerSm;
        if (e->gscratch.cap >= static_cast<size_t>(full) * per_warp) {
            // the scratch already holds every resident warp's table: no
            // cudaMemGetInfo (it can stall for tens of ms behind the driver)
            *warps = full;
            return ok();
        }
        static const size_t budget_max = [] {
            const char* v = getenv("MCMI_SCRATCH_GB");
            return (v && *v ? static_cast<size_t>(std::max(1, atoi(v))) : size_t{64}) << 30;
        }();
        size_t free_b = 0, total_b = 0;
        MCMI_TRY(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        const size_t budget = std::min<size_t>(budget_max, (free_b + e->gscratch.cap) / 2);
        int64_t w = std::min<int64_t>(static_cast<int64_t>(budget / per_warp), full);
        if (w < 1) return fail(MCMI_ENOMEM, "accumulator row too large for device memory");
        *warps = std::max<int64_t>(8, w / 8 * 8);
        return ok();
    };
    int64_t pool_used = 0;
    int cur = 0;
    unsigned long long total_steps = 0, total_deg = 0;
    // Runs `work` rows (row_list, or rows row_begin+offset ...) on tier t; returns
    // the number of rows that overflowed it (listed in ovf[cur] on return).
    auto run_tier = [&](const Tier& t, int64_t work, const int* row_list, int64_t offset,
                        int64_t* overflowed) -> Status {
        static const bool trace = getenv("MCMI_WALK_TRACE") != nullptr;
        const auto h0 = std::chrono::steady_clock::now();
        auto since = [&](std::chrono::steady_clock::time_point a) {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
        };
        const int64_t stride = stride_of(t);
        const int64_t need = pool_used + work * stride;
        MCMI_TRY(e->stage_col.grow_preserve(need * sizeof(int), pool_used * sizeof(int), s), "alloc staging");
        MCMI_TRY(e->stage_val.grow_preserve(need * sizeof(double), pool_used * sizeof(double), s),
                 "alloc staging");
        MCMI_TRY(cudaMemsetAsync(e->counters.p, 0, 8 * sizeof(unsigned long long), s), "memset");
        WalkArgs wa{};
        wa.t = Tables{n, e->rec.as<uint4>(), e->ent.as<double2>(), e->colA.as<int>(), e->b1.as<double>(), tri};
        wa.row_begin = row_begin;
        wa.row_list = row_list;
        wa.work_offset = offset;
        wa.n_work = work;
        {  // MCMI_WALK_CLAIM: rows per cursor claim (tuning); retries (row lists) claim one at a time
            static const int claim = [] {
                const char* v = getenv("MCMI_WALK_CLAIM");
                return v && *v ? std::max(1, std::min(64, atoi(v))) : 1;
            }();
            wa.claim_rows = row_list ? 1 : claim;
        }
        wa.n_chains = N;
        wa.max_len = std::clamp<int64_t>(L, 0, INT_MAX);  // walks beyond the log capacity overflow anyway
        wa.delta = cfg.delta;
        wa.seed = cfg.master_seed;
        wa.retain_k = cfg.retain_k;
        wa.rng_mode = cfg.rng_mode;
        wa.cap = t.cap;
        wa.cap_limit = t.cap_limit;
        wa.lanes = t.lanes;
        wa.log_stride = t.log_stride;
        wa.log_magic = static_cast<unsigned>((0x100000000ull + t.log_stride - 1) / t.log_stride);
        // reference stream: the first window's speculative stride.  Chains that
        // run to L draw L times (C5: every chain), so short walks start at L
        // (C5 10^2 x 8..64 -13..15% against 2); a row whose chains stop early
        // loses one window and goes dense.
        wa.ell0 = static_cast<int>(std::max<int64_t>(1, L <= 64 ? L : 2));
        wa.deg_stats = (cfg.flags & MCMI_FLAG_DEG_STATS) ? 1 : 0;
        wa.unscaled = (cfg.flags & MCMI_FLAG_UNSCALED) ? 1 : 0;
        // Neighbourhood slot tables (walk.cu, L = 2): their per-row set-up costs
        // about as much as a few thousand logged deposits, so they are used only
        // when a row logs many more deposits than its 2-hop neighbourhood holds
        // (C2 at eps = 0.01: 10976 vs 703, -1.6%; at the defaults, 282 deposits
        // per row, they cost C2 +60%, C3 +17%, C4 +14%).
        wa.nb_hint = (deposits >= 4096 && deposits / 12 >= reach) ? 1 : 0;
        wa.gscratch = nullptr;
        int64_t max_warps = 0;
        if (t.global) {
            Status gs = global_warps(t, &max_warps);
            if (gs.code) return gs;
            const size_t per_warp = walk_global_bytes_per_warp(t.cap, t.lanes, t.log_stride);
            MCMI_TRY(e->gscratch.ensure(static_cast<size_t>(max_warps) * per_warp), "alloc accumulator scratch");
            wa.gscratch = e->gscratch.as<unsigned char>();
        }
        wa.stage_col = e->stage_col.as<int>();
        wa.stage_val = e->stage_val.as<double>();
        wa.stage_base = pool_used;
        wa.stage_stride = stride;
        wa.row_cnt = e->row_cnt.as<int>();
        wa.row_src = e->row_src.as<int64_t>();
        wa.chains_used = e->chains_used.as<int64_t>();
        wa.entries_before = e->entries_before.as<int64_t>();
        wa.counters = e->counters.as<unsigned long long>();
        wa.overflow_list = e->ovf[cur].as<int>();
        const double setup_ms = trace ? since(h0) : 0.0;
        const auto h1 = std::chrono::steady_clock::now();
        MCMI_TRY(cudaEventRecord(e->ev[4], s), "cudaEventRecord");
        MCMI_TRY(launch_walk(wa, t.warps_per_block, e->num_sms, t.global, max_warps, s), "walk kernel");
        MCMI_TRY(cudaEventRecord(e->ev[5], s), "cudaEventRecord");
        st.launches += 1;
        MCMI_TRY(cudaMemcpyAsync(e->h_ctr, e->counters.p, 8 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s),
                 "read counters");
        MCMI_TRY(cudaStreamSynchronize(s), "walk kernel");
        float tw = 0;
        cudaEventElapsedTime(&tw, e->ev[4], e->ev[5]);
        st.ms_walk_kernel += tw;
        if (trace)  // MCMI_WALK_TRACE=1: host setup / launch-to-sync wall / kernel device time per tier launch
            std::fprintf(stderr, "mcmi walk: cap %d%s rows %lld setup %.2f ms wall %.2f ms kernel %.2f ms\n", t.cap,
                         t.global ? " (global)" : "", static_cast<long long>(work), setup_ms, since(h1), tw);
        total_steps += e->h_ctr[1];
        total_deg += e->h_ctr[2];
        pool_used += work * stride;
        *overflowed = static_cast<int64_t>(e->h_ctr[3]);
        return ok();
    };

    // Pilot: when rows may overflow the first tier, build the first rows on the
    // last tier (which cannot overflow: its cap_limit >= bound), and start the
    // rest on the tier a cost model picks from the pilot rows' distinct-column
    // counts.  Rows the pilot under-estimates still overflow into the next
    // tiers, so results never depend on this choice.
    size_t t0 = 0;
    int64_t pilot_rows = 0;
    int64_t pilot = std::min<int64_t>(1024, rows / 4);
    if (tiers.size() > 1 && deposits >= kLongRowDeposits && tiers.back().global) {
        // Long rows (C5's wide corners: a row is 10^5+ steps of one warp): a
        // launch lasts a whole number of row latencies (waves of W resident
        // warps) however few rows its last wave holds.  All rows in one wave
        // when they fit (10^5 x 64: 2 launches -> 1); otherwise the pilot
        // fills up to a wave, at most a quarter of the rows (10^4 x 32: 4 row
        // latencies -> 3; 10^4 x 16: 563 -> 521 ms against a 1024-row pilot).
        int64_t w = 0;
        Status gs = global_warps(tiers.back(), &w);
        if (gs.code) return gs;
        pilot = rows <= w ? rows : std::max(pilot, std::min(rows / 4, w));
        // the pilot's output stays staged until its chunk is assembled
        const int64_t staged = staging_budget_bytes() / (stride_of(tiers.back()) * 12);
        pilot = std::max<int64_t>(std::min<int64_t>(1024, rows / 4), std::min(pilot, staged));
    }
    if (tiers.size() > 1 && pilot >= 64) {
        int64_t ovf = 0;
        Status ps = run_tier(tiers.back(), pilot, nullptr, 0, &ovf);
        if (ps.code) return ps;
        if (ovf != 0)
            return fail(MCMI_ENOMEM, std::to_string(ovf) +
                                         " rows overflowed every accumulator tier (more distinct columns than "
                                         "device memory allows, or walks longer than 65536 steps)");
        if (!e->h_pilot_buf(static_cast<size_t>(pilot))) return fail(MCMI_ENOMEM, "cudaMallocHost (pilot)");
        MCMI_TRY(cudaMemcpyAsync(e->h_pilot, e->entries_before.p, pilot * sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, s),
                 "read pilot");
        MCMI_TRY(cudaStreamSynchronize(s), "read pilot");
        // A row of s distinct columns costs c_t on the tier that holds it and
        // ~c_t * limit_t / s on each tier it overflows first (it aborts once the
        // table is full).  Relative costs (measured on the C5 grid,
        // tools/c5_sweep.py): shared memory (<= 256 slots, 48 warps/SM) 1, the
        // 1024-slot global-scratch tier 2, larger global tables 3.
        auto tier_cost = [](const Tier& t) { return t.global ? (t.cap <= 1024 ? 2.0 : 3.0) : 1.0; };
        double best = 0.0;
        for (size_t c0 = 0; c0 < tiers.size(); ++c0) {
            double cost = 0.0;
            for (int64_t i = 0; i < pilot; ++i) {
                const double sr = static_cast<double>(std::max<int64_t>(1, e->h_pilot[i]));
                for (size_t t = c0; t < tiers.size(); ++t) {
                    if (tiers[t].cap_limit >= e->h_pilot[i] || t + 1 == tiers.size()) {
                        cost += tier_cost(tiers[t]);
                        break;
                    }
                    cost += tier_cost(tiers[t]) * std::min(1.0, tiers[t].cap_limit / sr);
                }
            }
            if (c0 == 0 || cost < best) {
                best = cost;
                t0 = c0;
            }
        }
        st.hash_cap = tiers[t0].cap;
        pilot_rows = pilot;
    }
    // Walks rows [lo, hi) (local) starting on tier t0, retrying overflows.
    auto walk_rows = [&](int64_t lo, int64_t hi) -> Status {
        int64_t work = hi - lo;
        const int* row_list = nullptr;
        for (size_t ti = t0; ti < tiers.size() && work > 0; ++ti) {
            int64_t overflowed = 0;
            Status ts = run_tier(tiers[ti], work, row_list, row_list ? 0 : lo, &overflowed);
            if (ts.code) return ts;
            if (ti > t0) st.rows_retried += work;
            work = overflowed;
            row_list = e->ovf[cur].as<int>();
            cur ^= 1;
        }
        if (work > 0)
            return fail(MCMI_ENOMEM, std::to_string(work) +
                                         " rows overflowed every accumulator tier (more distinct columns than "
                                         "device memory allows, or walks longer than 65536 steps)");
        return ok();
    };

    // ---- rows in chunks, each walked, scanned and compacted in row order
    // (mc_engine.cpp:207-225).  Device output (no sink): one chunk unless
    // rows x slot stride exceeds the staging budget; entries are appended to the
    // engine's output buffers.  Host sink: chunk sizes fall geometrically (few
    // chunk boundaries, each costs the walk kernel's tail, and a small last
    // chunk, whose copy is the exposed one); chunk c's device->host copy (copy
    // stream) overlaps chunk c+1's walk, through double-buffered device slabs.
    // MCMI_STREAM_CHUNKS / MCMI_STREAM_RATIO: tuning overrides.
    const int64_t entry_bytes = static_cast<int64_t>(sizeof(int) + sizeof(double));
    const int64_t budget_rows =
        std::max<int64_t>(pilot_rows + 1, staging_budget_bytes() / (stride_of(tiers[t0]) * entry_bytes));
    std::vector<int64_t> bnd{0};
    if (!sink) {
        const int64_t nch = std::max<int64_t>(1, (rows + budget_rows - 1) / budget_rows);
        for (int64_t c = 1; c <= nch; ++c) bnd.push_back(std::max(bnd.back(), rows * c / nch));
    } else {
        int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(8, rows / 65536));
        double ratio = 0.65;
        if (const char* v = getenv("MCMI_STREAM_CHUNKS")) nchunk = std::max<int64_t>(1, std::min<int64_t>(64, atoll(v)));
        if (const char* v = getenv("MCMI_STREAM_RATIO")) ratio = std::max(0.05, std::min(1.0, atof(v)));
        nchunk = std::min<int64_t>(nchunk, std::max<int64_t>(rows, 1));
        int64_t start = 0;
        if (sink->first_chunk > 0.0 && nchunk > 1) {  // a small first chunk: an early entry-count estimate
            start = std::max<int64_t>(1, static_cast<int64_t>(static_cast<double>(rows) * sink->first_chunk));
            bnd.push_back(start);
            --nchunk;
        }
        double wsum = 0.0, w = 1.0;
        for (int64_t c = 0; c < nchunk; ++c, w *= ratio) wsum += w;
        double acc = 0.0;
        w = 1.0;
        for (int64_t c = 1; c < nchunk; ++c, w *= ratio) {
            acc += w;
            bnd.push_back(std::max(bnd.back() + 1,
                                   start + static_cast<int64_t>(static_cast<double>(rows - start) * acc / wsum)));
        }
        bnd.push_back(rows);
        // no chunk larger than the staging budget
        std::vector<int64_t> split{0};
        for (size_t c = 1; c < bnd.size(); ++c)
            for (int64_t x = split.back(); x < bnd[c];) split.push_back(x = std::min(bnd[c], x + budget_rows));
        bnd.swap(split);
    }
    if (bnd.size() > 1 && bnd[1] < pilot_rows) bnd[1] = pilot_rows;  // chunk 0 holds the pilot rows
    for (size_t c = 1; c < bnd.size(); ++c) bnd[c] = std::min(rows, std::max(bnd[c], bnd[c - 1]));
    const int64_t nchunk = static_cast<int64_t>(bnd.size()) - 1;

    MCMI_TRY(e->out_rp.ensure((rows + 1) * sizeof(int64_t)), "alloc row_ptr");
    if (sink) {
        MCMI_TRY(e->ensure_copy_stream(), "copy stream");
        MCMI_TRY(cudaStreamSynchronize(e->copy), "drain copies");
    }
    // every exit (errors included) waits for the queued copies into the sink
    struct CopyDrain {
        cudaStream_t s;
        ~CopyDrain() {
            if (s) cudaStreamSynchronize(s);
        }
    } drain{sink ? e->copy : nullptr};
    int64_t slab_cap = static_cast<int64_t>(std::min(e->col_slab[0].cap / sizeof(int64_t),
                                                     e->val_slab[0].cap / sizeof(double)));
    int64_t running = 0;
    bool fits = true;
    // MCMI_STREAM_DEBUG=1: per-chunk device timestamps of walk and copy
    const bool dbg = sink && getenv("MCMI_STREAM_DEBUG") != nullptr;
    std::vector<cudaEvent_t> dev(dbg ? 4 * nchunk : 0);
    for (auto& ev : dev) cudaEventCreate(&ev);
    for (int64_t c = 0; c < nchunk; ++c) {
        const int64_t lo = bnd[c], hi = bnd[c + 1];  // empty only when rows == 0 (the scan writes row_ptr[0])
        if (dbg) cudaEventRecord(dev[4 * c], s);
        if (c > 0) pool_used = 0;  // staging reused per chunk (chunk 0 keeps the pilot rows' slots)
        Status ws = walk_rows(c == 0 ? pilot_rows : lo, hi);
        if (ws.code) return ws;
        if (c + 1 == nchunk) MCMI_TRY(cudaEventRecord(e->ev[2], s), "cudaEventRecord");
        if (dbg) cudaEventRecord(dev[4 * c + 1], s);
        const int64_t cr = hi - lo;
        int64_t* rp_chunk = e->out_rp.as<int64_t>() + lo;  // chunk-local offsets, then global
        // (host sink) wait until chunk c-2's copies released this slab pair
        if (sink) MCMI_TRY(cudaStreamWaitEvent(s, e->copy_done[c & 1], 0), "wait copy");
        MCMI_TRY(scan_rows_exclusive(e->row_cnt.as<int>() + lo, rp_chunk, cr, e->scan_tmp.p, s), "scan rows");
        MCMI_TRY(cudaMemcpyAsync(e->h_i64, rp_chunk + cr, sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                 "read chunk nnz");
        MCMI_TRY(cudaStreamSynchronize(s), "scan rows");
        const int64_t cn = e->h_i64[0];
        st.launches += (cr > 0 ? 3 : 1);
        if (!sink) {
            const int64_t need = std::max<int64_t>(running + cn, 1);
            MCMI_TRY(running ? e->out_col.grow_preserve(need * sizeof(int64_t), running * sizeof(int64_t), s)
                             : e->out_col.ensure(need * sizeof(int64_t)),
                     "alloc col");
            MCMI_TRY(running ? e->out_val.grow_preserve(need * sizeof(double), running * sizeof(double), s)
                             : e->out_val.ensure(need * sizeof(double)),
                     "alloc val");
            MCMI_TRY(launch_compact(e->stage_col.as<int>(), e->stage_val.as<double>(), e->row_src.as<int64_t>() + lo,
                                    e->row_cnt.as<int>() + lo, rp_chunk, cr, e->out_col.as<int64_t>() + running,
                                    e->out_val.as<double>() + running, s),
                     "compact");
            st.launches += (cr > 0 ? 1 : 0);
            if (running) {  // cr + 1: the chunk's end entry is the running total (row_ptr[rows] at the end)
                MCMI_TRY(launch_add_offset(rp_chunk, running, cr + 1, s), "row_ptr offset");
                st.launches += 1;
            }
        } else {
            if (fits && running + cn > sink->capacity && sink->grow) {
                MCMI_TRY(cudaStreamSynchronize(e->copy), "drain copies");  // nothing in flight into the old buffer
                const double done = static_cast<double>(std::max<int64_t>(hi, 1));
                const int64_t est = static_cast<int64_t>(static_cast<double>(running + cn) * rows / done * 1.06) + 1024;
                Status gs = sink->grow(*sink, running + cn, std::max(est, running + cn), running);
                if (gs.code) return gs;
            }
            if (running + cn > sink->capacity) fits = false;
            if (fits) {
                if (cn > slab_cap) {
                    MCMI_TRY(cudaStreamSynchronize(e->copy), "drain copies");
                    for (int q = 0; q < 2; ++q) {
                        MCMI_TRY(e->col_slab[q].ensure(std::max<int64_t>(cn, 1) * sizeof(int64_t)), "alloc slab");
                        MCMI_TRY(e->val_slab[q].ensure(std::max<int64_t>(cn, 1) * sizeof(double)), "alloc slab");
                    }
                    slab_cap = cn;
                }
                int64_t* cs = e->col_slab[c & 1].as<int64_t>();
                double* vs = e->val_slab[c & 1].as<double>();
                MCMI_TRY(launch_compact(e->stage_col.as<int>(), e->stage_val.as<double>(),
                                        e->row_src.as<int64_t>() + lo, e->row_cnt.as<int>() + lo, rp_chunk, cr, cs,
                                        vs, s),
                         "compact");
                MCMI_TRY(launch_add_offset(rp_chunk, running, cr, s), "row_ptr offset");
                MCMI_TRY(cudaEventRecord(e->chunk_ready, s), "cudaEventRecord");
                MCMI_TRY(cudaStreamWaitEvent(e->copy, e->chunk_ready, 0), "wait chunk");
                if (dbg) cudaEventRecord(dev[4 * c + 2], e->copy);
                auto d2h = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
                    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, e->copy) : cudaSuccess;
                };
                MCMI_TRY(d2h(sink->col_idx + running, cs, cn * sizeof(int64_t)), "D2H col");
                MCMI_TRY(d2h(sink->values + running, vs, cn * sizeof(double)), "D2H val");
                MCMI_TRY(cudaEventRecord(e->copy_done[c & 1], e->copy), "cudaEventRecord");
                if (dbg) cudaEventRecord(dev[4 * c + 3], e->copy);
                if (sink->queued) sink->queued(running, running + cn, e->copy);
                st.launches += 2;
            }
        }
        running += cn;
        if (sink && sink->progress) sink->progress(hi, running, rows);
    }
    const int64_t out_nnz = running;
    if (!sink) {
        MCMI_TRY(e->out_col.ensure(sizeof(int64_t)), "alloc col");  // valid pointers for empty results
        MCMI_TRY(e->out_val.ensure(sizeof(double)), "alloc val");
    } else {
        MCMI_TRY(cudaStreamSynchronize(e->copy), "D2H");
        if (dbg) {
            for (int64_t c = 0; c < nchunk; ++c) {
                float w0 = 0, w1 = 0, c0 = 0, c1 = 0;
                cudaEventElapsedTime(&w0, e->ev[0], dev[4 * c]);
                cudaEventElapsedTime(&w1, e->ev[0], dev[4 * c + 1]);
                cudaEventElapsedTime(&c0, e->ev[0], dev[4 * c + 2]);
                cudaEventElapsedTime(&c1, e->ev[0], dev[4 * c + 3]);
                fprintf(stderr, "chunk %lld walk %.2f-%.2f copy %.2f-%.2f ms\n", static_cast<long long>(c), w0, w1,
                        c0, c1);
            }
        }
        if (fits) {  // row pointers and RowMeta: one copy each, after the walks
            auto cp = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
                return (dst && bytes) ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s) : cudaSuccess;
            };
            MCMI_TRY(cp(sink->row_ptr, e->out_rp.p, rows * sizeof(int64_t)), "D2H row_ptr");
            MCMI_TRY(cp(sink->chains_used, e->chains_used.p, rows * sizeof(int64_t)), "D2H meta");
            MCMI_TRY(cp(sink->entries_before, e->entries_before.p, rows * sizeof(int64_t)), "D2H meta");
            MCMI_TRY(cudaStreamSynchronize(s), "D2H row_ptr");
            sink->row_ptr[rows] = running;
        }
        if (!fits) {
            st.nnz = out_nnz;
            if (stats) *stats = st;
            return fail(MCMI_ENOMEM, "output capacity " + std::to_string(sink->capacity) + " < nnz " +
                                         std::to_string(out_nnz));
        }
    }
    for (auto& ev : dev) cudaEventDestroy(ev);
    st.walk_steps = static_cast<int64_t>(total_steps);
    st.walk_deg_sum = (cfg.flags & MCMI_FLAG_DEG_STATS) ? static_cast<int64_t>(total_deg) : -1;
    MCMI_TRY(cudaEventRecord(e->ev[3], s), "cudaEventRecord");
    MCMI_TRY(cudaStreamSynchronize(s), "assembly");
    float t01 = 0, t12 = 0, t23 = 0, t03 = 0;
    cudaEventElapsedTime(&t01, e->ev[0], e->ev[1]);
    cudaEventElapsedTime(&t12, e->ev[1], e->ev[2]);
    cudaEventElapsedTime(&t23, e->ev[2], e->ev[3]);
    cudaEventElapsedTime(&t03, e->ev[0], e->ev[3]);
    st.ms_tables = t01;
    st.ms_walk = t12;
    st.ms_assemble = t23;
    st.ms_total = t03;
    st.nnz = out_nnz;

    out->row_begin = row_begin;
    out->row_end = row_end;
    out->nnz = out_nnz;
    out->row_ptr = e->out_rp.as<int64_t>();
    out->col_idx = e->out_col.as<int64_t>();
    out->values = e->out_val.as<double>();
    out->chains_used = e->chains_used.as<int64_t>();
    out->entries_before = e->entries_before.as<int64_t>();
    if (stats) *stats = st;
    return ok();
}

// One cached engine per device for the host API (buffers reused across calls).
std::mutex g_cache_mu;
std::vector<mcmi_engine*> g_cache;  // idle engines

mcmi_engine* acquire_engine(int device, Status* st) {
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (size_t i = 0; i < g_cache.size(); ++i)
            if (g_cache[i]->device == device) {
                mcmi_engine* e = g_cache[i];
                g_cache.erase(g_cache.begin() + static_cast<long>(i));
                return e;
            }
    }
    auto* e = new mcmi_engine();
    *st = engine_init(e, device);
    if (st->code) {
        engine_release(e);
        delete e;
        return nullptr;
    }
    return e;
}

void release_engine(mcmi_engine* e) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.push_back(e);
}

// Host CSR in: stage B on the engine's stream (stream-ordered pool allocations,
// cached across calls), build rows [row_begin, row_end), release the staging.
Status build_from_host(mcmi_engine* e, const mcmi_csr_view& b, const mcmi_config& cfg, int64_t row_begin,
                       int64_t row_end, mcmi_device_csr* dc, mcmi_stats* stats, HostSink* sink,
                       const ApSource* ap_host = nullptr) {
    const int64_t n = b.n;
    if (n < 0) return fail(MCMI_EINVAL, "negative dimension");
    if (n > 0 && !b.row_ptr) return fail(MCMI_EINVAL, "null row_ptr");
    const int64_t nnz = n > 0 ? b.row_ptr[n] : 0;
    if (nnz < 0) return fail(MCMI_EINVAL, "row_ptr[n] is negative");
    if (nnz > 0 && (!b.col_idx || !b.values)) return fail(MCMI_EINVAL, "null col_idx / values");
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    void *d_rp = nullptr, *d_ci = nullptr, *d_v = nullptr, *d_p = nullptr;
    if (ap_host) MCMI_TRY(cudaMallocAsync(&d_p, std::max<int64_t>(nnz, 1) * sizeof(double), s), "alloc P");
    MCMI_TRY(cudaMallocAsync(&d_rp, (n + 1) * sizeof(int64_t), s), "alloc B");
    MCMI_TRY(cudaMallocAsync(&d_ci, std::max<int64_t>(nnz, 1) * sizeof(int64_t), s), "alloc B");
    MCMI_TRY(cudaMallocAsync(&d_v, std::max<int64_t>(nnz, 1) * sizeof(double), s), "alloc B");
    Status st;
    // pageable inputs (a reference caller's std::vector) go through pinned
    // bounce buffers in one pipeline: 11 GB/s -> ~40 GB/s on the box (hostio.h)
    const auto hs0 = std::chrono::steady_clock::now();
    {
        const H2DSegment segs[4] = {{d_rp, b.row_ptr, static_cast<size_t>(n + 1) * sizeof(int64_t)},
                                    {d_ci, b.col_idx, static_cast<size_t>(nnz) * sizeof(int64_t)},
                                    {d_v, b.values, static_cast<size_t>(nnz) * sizeof(double)},
                                    {d_p, ap_host ? ap_host->p_values : nullptr,
                                     ap_host ? static_cast<size_t>(nnz) * sizeof(double) : 0}};
        st = cuda_status(stage_h2d(segs, 4, s), "H2D");
    }
    if (getenv("MCMI_STREAM_DEBUG"))
        std::fprintf(stderr, "mcmi stage B: %.2f ms host (%lld bytes)\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - hs0).count(),
                     static_cast<long long>((n + 1 + 2 * nnz) * 8));
    if (st.code == MCMI_OK) {
        const mcmi_csr_view dv{n, static_cast<int64_t*>(d_rp), static_cast<int64_t*>(d_ci),
                               static_cast<double*>(d_v)};
        ApSource ap_dev{static_cast<const double*>(d_p), ap_host ? ap_host->n_chains : 0,
                        ap_host ? ap_host->max_len : 0};
        st = engine_build(e, dv, cfg, row_begin, row_end, s, dc, stats, sink, ap_host ? &ap_dev : nullptr);
    }
    if (d_p) cudaFreeAsync(d_p, s);
    cudaFreeAsync(d_rp, s);
    cudaFreeAsync(d_ci, s);
    cudaFreeAsync(d_v, s);
    return st;
}

}  // namespace

// One device shard of a multi-GPU host build: the arrays are the engine's own
// output buffers (no per-call device allocation or free); the parts keep their
// engines checked out of the cache until they are copied out and freed.
struct ResultPart {
    mcmi_engine* engine = nullptr;
    int64_t rows = 0, nnz = 0;
    const int64_t* rp = nullptr;
    const int64_t* ci = nullptr;
    const double* v = nullptr;
    const int64_t* cu = nullptr;
    const int64_t* eb = nullptr;
};

struct DeviceParts {
    int64_t n = 0, nnz = 0;
    int64_t n_chains = 1, max_len = 1;
    mcmi_stats stats{};
    std::vector<ResultPart> parts;  // row blocks in row order (one per GPU)
};

// Host-resident result of mcmi_build* / mcmi_job_*: library-owned page-locked
// arrays (pooled across builds, hostio.h), filled while the walks run.
struct mcmi_result {
    int64_t n = 0, nnz = 0;
    int64_t n_chains = 1, max_len = 1;
    mcmi_stats stats{};
    PinnedBuf rp, ci, v, cu, eb;
    ~mcmi_result() {
        for (PinnedBuf* b : {&rp, &ci, &v, &cu, &eb}) pinned_release(*b);
    }
};

// A host build running on a library thread (mcmi_build_start).  Once the
// caller attaches its own entry arrays (mcmi_job_attach), a copier thread
// moves every row chunk from the library's page-locked result into them as
// soon as the chunk's device->host copy has completed, while later chunks are
// still walking; mcmi_job_finish reports how many leading entries arrived.
struct mcmi_job {
    mcmi_csr_view b{};
    mcmi_config cfg{};
    int64_t lo = 0, hi = -1;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    bool has_estimate = false, done = false;
    int64_t estimate = -1;
    int code = MCMI_OK;
    std::string msg;
    mcmi_result* result = nullptr;
    // progressive delivery (guarded by mu)
    struct Range {
        int64_t lo, hi;
        cudaEvent_t ev;
    };
    std::deque<Range> landed;       // queued chunk copies (device -> page-locked), in entry order
    int64_t landed_hi = 0;          // entries [0, landed_hi) are in the result's host arrays
    std::thread copier;
    bool build_over = false;        // no more ranges will be queued
    bool growing = false, busy = false;
    int64_t* dst_col = nullptr;
    double* dst_val = nullptr;
    int64_t dst_cap = 0;            // entries [0, dst_cap) of the attached arrays may be written
    int64_t delivered = 0;          // entries [0, delivered) are in the attached arrays
    const int64_t* src_col = nullptr;  // the result's current page-locked arrays
    const double* src_val = nullptr;

    int64_t deliverable() const { return dst_col ? std::min(landed_hi, dst_cap) : 0; }
    void copier_loop() {
        for (;;) {
            cudaEvent_t ev = nullptr;
            int64_t rhi = 0, a0 = 0, a1 = 0;
            const int64_t* sc = nullptr;
            const double* sv = nullptr;
            int64_t* dc = nullptr;
            double* dv = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] {
                    return !growing && (!landed.empty() || delivered < deliverable() || build_over);
                });
                if (!landed.empty()) {
                    ev = landed.front().ev;
                    rhi = landed.front().hi;
                    landed.pop_front();
                } else if (delivered < deliverable()) {
                    a0 = delivered;
                    a1 = deliverable();
                    busy = true;
                    sc = src_col;
                    sv = src_val;
                    dc = dst_col;
                    dv = dst_val;
                } else {
                    return;  // the build is over and everything landed so far is delivered
                }
            }
            if (ev) {  // a chunk's device->host copy: wait for it, then it is deliverable
                const bool ok = cudaEventSynchronize(ev) == cudaSuccess;
                cudaEventDestroy(ev);
                std::lock_guard<std::mutex> lk(mu);
                if (ok) landed_hi = std::max(landed_hi, rhi);
                cv.notify_all();
                continue;
            }
            parallel_copy(dc + a0, sc + a0, static_cast<size_t>(a1 - a0) * sizeof(int64_t));
            parallel_copy(dv + a0, sv + a0, static_cast<size_t>(a1 - a0) * sizeof(double));
            std::lock_guard<std::mutex> lk(mu);
            delivered = a1;
            busy = false;
            cv.notify_all();
        }
    }
    // the build thread is about to re-point the result's arrays: wait for the copier
    void pause_copier() {
        std::unique_lock<std::mutex> lk(mu);
        growing = true;
        cv.wait(lk, [&] { return !busy; });
    }
    void resume_copier(const int64_t* c, const double* v) {
        std::lock_guard<std::mutex> lk(mu);
        src_col = c;
        src_val = v;
        growing = false;
        cv.notify_all();
    }
};

namespace {

// Devices of a build: cfg.n_gpus (0 = env MCMI_GPUS, else 1) consecutive
// ordinals from cfg.device.  MCMI_SHARD_WRAP=1 maps ordinals modulo the
// visible device count (several shards per GPU: a test hook for one-GPU boxes).
Status shard_devices(const mcmi_config& cfg, std::vector<int>* devs) {
    int g = cfg.n_gpus;
    if (g <= 0) {
        const char* env = std::getenv("MCMI_GPUS");
        g = env && *env ? std::atoi(env) : 1;
        if (g <= 0) g = 1;
    }
    devs->clear();
    if (g == 1) {
        devs->push_back(cfg.device);
        return ok();
    }
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
        cudaGetLastError();
        return fail(MCMI_ENODEV, "no CUDA device");
    }
    const char* wrap = std::getenv("MCMI_SHARD_WRAP");
    const bool wrapped = wrap && *wrap && std::strcmp(wrap, "0") != 0;
    for (int i = 0; i < g; ++i) {
        const int d = cfg.device + i;
        if (d >= count && !wrapped)
            return fail(MCMI_ENODEV, "n_gpus=" + std::to_string(g) + " needs devices " + std::to_string(cfg.device) +
                                         ".." + std::to_string(cfg.device + g - 1) + " but " +
                                         std::to_string(count) + " are visible");
        devs->push_back(d % count);
    }
    return ok();
}

// Contiguous row blocks of [lo, hi) balanced on cost(r) = 1 + nnz(r): block g
// starts at the first row whose cost prefix reaches total * g / G (the same
// edges as distributed.partition_rows).
std::vector<int64_t> partition_rows(const int64_t* rp, int64_t lo, int64_t hi, int g) {
    std::vector<int64_t> edges(static_cast<size_t>(g) + 1, lo);
    edges[g] = hi;
    if (hi <= lo) return edges;
    auto cost = [&](int64_t i) { return static_cast<double>(i - lo) + static_cast<double>(rp[i] - rp[lo]); };
    const double total = cost(hi);
    for (int k = 1; k < g; ++k) {
        const double target = total * k / g;
        int64_t a = lo, b = hi + 1;  // first i in [lo, hi] with cost(i) >= target
        while (a < b) {
            const int64_t m = a + (b - a) / 2;
            if (cost(m) < target) a = m + 1;
            else b = m;
        }
        edges[k] = std::max(std::min(a, hi), edges[k - 1]);
    }
    return edges;
}

// Builds rows [lo, hi) on every device of the build, one host thread per
// shard (each stages B on its own GPU); rows are independent
// (mc_engine.cpp:164-178), so the row-ordered concatenation of the shards is
// the single-GPU M.  On success the result owns the engines.
Status build_parts(const mcmi_csr_view& b, const mcmi_config& cfg, int64_t lo, int64_t hi, DeviceParts* r) {
    std::vector<int> devs;
    if (Status st = shard_devices(cfg, &devs); st.code) return st;
    const int64_t n = b.n;
    if (lo < 0) lo = 0;
    if (hi < 0 || hi > n) hi = n;
    if (hi < lo) hi = lo;
    const int g = static_cast<int>(devs.size());
    if (g > 1 && n > 0 && !b.row_ptr) return fail(MCMI_EINVAL, "null row_ptr");
    const std::vector<int64_t> edges = g > 1 ? partition_rows(b.row_ptr, lo, hi, g) : std::vector<int64_t>{lo, hi};
    struct Job {
        mcmi_engine* e = nullptr;
        mcmi_device_csr dc{};
        mcmi_stats st{};
        Status status;
    };
    std::vector<Job> jobs(static_cast<size_t>(g));
    auto run = [&](int i) {
        Job& j = jobs[static_cast<size_t>(i)];
        j.e = acquire_engine(devs[static_cast<size_t>(i)], &j.status);
        if (!j.e) return;
        mcmi_config c = cfg;
        c.device = devs[static_cast<size_t>(i)];
        j.status = build_from_host(j.e, b, c, edges[i], edges[i + 1], &j.dc, &j.st, nullptr);
    };
    if (g == 1) {
        run(0);
    } else {
        std::vector<std::thread> threads;
        for (int i = 0; i < g; ++i) threads.emplace_back(run, i);
        for (auto& t : threads) t.join();
    }
    Status first;
    for (auto& j : jobs)
        if (j.status.code && !first.code) first = j.status;
    if (first.code) {
        for (auto& j : jobs)
            if (j.e) release_engine(j.e);
        return first;
    }
    r->n = hi - lo;
    r->nnz = 0;
    mcmi_stats& t = r->stats;
    t = jobs[0].st;
    for (size_t i = 0; i < jobs.size(); ++i) {
        const Job& j = jobs[i];
        ResultPart p;
        p.engine = j.e;
        p.rows = j.dc.row_end - j.dc.row_begin;
        p.nnz = j.dc.nnz;
        p.rp = j.dc.row_ptr;
        p.ci = j.dc.col_idx;
        p.v = j.dc.values;
        p.cu = j.dc.chains_used;
        p.eb = j.dc.entries_before;
        r->parts.push_back(p);
        r->nnz += p.nnz;
        if (i == 0) continue;
        t.rows += j.st.rows;
        t.nnz += j.st.nnz;
        t.walk_steps += j.st.walk_steps;
        if (t.walk_deg_sum >= 0 && j.st.walk_deg_sum >= 0) t.walk_deg_sum += j.st.walk_deg_sum;
        t.rows_retried += j.st.rows_retried;
        t.launches += j.st.launches;
        t.hash_cap = std::max(t.hash_cap, j.st.hash_cap);
        // device times: the shards run concurrently, the build takes the slowest
        t.ms_tables = std::max(t.ms_tables, j.st.ms_tables);
        t.ms_walk = std::max(t.ms_walk, j.st.ms_walk);
        t.ms_assemble = std::max(t.ms_assemble, j.st.ms_assemble);
        t.ms_total = std::max(t.ms_total, j.st.ms_total);
        t.ms_walk_kernel = std::max(t.ms_walk_kernel, j.st.ms_walk_kernel);
    }
    r->n_chains = t.n_chains;
    r->max_len = t.max_len;
    return ok();
}

// Copies the parts to their global offsets in the caller's arrays (any pointer
// may be NULL): every GPU's device->host copy is in flight at once, then the
// shard-local row pointers are shifted by the entries of the shards before.
int copy_parts(const DeviceParts* r, int64_t* row_ptr, int64_t* col_idx, double* values, int64_t* chains_used,
               int64_t* entries_before) {
    cudaError_t e = cudaSuccess;
    int64_t row_off = 0, nnz_off = 0;
    for (const ResultPart& p : r->parts) {
        if (e == cudaSuccess) e = cudaSetDevice(p.engine->device);
        cudaStream_t s = p.engine->own;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            if (dst && src && bytes && e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s);
        };
        cp(col_idx ? col_idx + nnz_off : nullptr, p.ci, p.nnz * sizeof(int64_t));  // largest first
        cp(values ? values + nnz_off : nullptr, p.v, p.nnz * sizeof(double));
        cp(row_ptr ? row_ptr + row_off : nullptr, p.rp, p.rows * sizeof(int64_t));  // row_ptr[n] is set below
        cp(chains_used ? chains_used + row_off : nullptr, p.cu, p.rows * sizeof(int64_t));
        cp(entries_before ? entries_before + row_off : nullptr, p.eb, p.rows * sizeof(int64_t));
        row_off += p.rows;
        nnz_off += p.nnz;
    }
    for (const ResultPart& p : r->parts) {
        if (e == cudaSuccess) e = cudaSetDevice(p.engine->device);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p.engine->own);
    }
    if (e != cudaSuccess) return MCMI_ECUDA;
    if (row_ptr) {
        row_off = nnz_off = 0;
        for (const ResultPart& p : r->parts) {
            if (nnz_off)
                for (int64_t i = 0; i < p.rows; ++i) row_ptr[row_off + i] += nnz_off;
            row_off += p.rows;
            nnz_off += p.nnz;
        }
        row_ptr[row_off] = nnz_off;
    }
    return MCMI_OK;
}

void free_parts(DeviceParts* r) {
    for (ResultPart& p : r->parts)
        if (p.engine) release_engine(p.engine);
    r->parts.clear();
}

// The host drop-in's build of rows [lo, hi) into a host-resident result.  One
// GPU: the streamed build (row chunks copied to pinned memory while the next
// chunk walks); the entry arrays are sized from the first chunks' counts
// (`on_estimate` receives that extrapolation, or the exact count) and grow if
// later chunks need more.  Several GPUs (cfg.n_gpus): concurrent row blocks,
// then every GPU's shard copied to its global offset.
Status build_host(const mcmi_csr_view& b, const mcmi_config& cfg, int64_t lo, int64_t hi, mcmi_result* r,
                  const std::function<void(int64_t)>& on_estimate, double first_chunk,
                  const ApSource* ap_host = nullptr, mcmi_job* job = nullptr) {
    std::vector<int> devs;
    if (Status st = shard_devices(cfg, &devs); st.code) return st;
    const int64_t n = b.n;
    if (n < 0) return fail(MCMI_EINVAL, "negative dimension");
    if (lo < 0) lo = 0;
    if (hi < 0 || hi > n) hi = n;
    if (hi < lo) hi = lo;
    const int64_t rows = hi - lo;
    auto need = [](PinnedBuf& buf, int64_t count) -> bool {
        buf = pinned_acquire(static_cast<size_t>(std::max<int64_t>(count, 1)) * 8);
        return buf.p != nullptr;
    };
    if (devs.size() > 1 && !ap_host) {
        DeviceParts dp;
        if (Status st = build_parts(b, cfg, lo, hi, &dp); st.code) return st;
        if (on_estimate) on_estimate(dp.nnz);
        Status st;
        if (!need(r->rp, rows + 1) || !need(r->ci, dp.nnz) || !need(r->v, dp.nnz) || !need(r->cu, rows) ||
            !need(r->eb, rows)) {
            st = fail(MCMI_ENOMEM, "cudaHostAlloc of the result failed");
        } else if (const int code = copy_parts(&dp, r->rp.as<int64_t>(), r->ci.as<int64_t>(), r->v.as<double>(),
                                               r->cu.as<int64_t>(), r->eb.as<int64_t>());
                   code) {
            st = fail(code, "device->host copy failed");
        }
        r->n = dp.n;
        r->nnz = dp.nnz;
        r->n_chains = dp.n_chains;
        r->max_len = dp.max_len;
        r->stats = dp.stats;
        free_parts(&dp);
        return st;
    }
    mcmi_config c = cfg;
    c.device = devs[0];
    Status st;
    mcmi_engine* e = acquire_engine(c.device, &st);
    if (!e) return st;
    if (!need(r->rp, rows + 1) || !need(r->cu, rows) || !need(r->eb, rows)) {
        release_engine(e);
        return fail(MCMI_ENOMEM, "cudaHostAlloc of the result failed");
    }
    HostSink sink;
    sink.row_ptr = r->rp.as<int64_t>();
    sink.chains_used = r->cu.as<int64_t>();
    sink.entries_before = r->eb.as<int64_t>();
    sink.first_chunk = first_chunk;
    sink.grow = [r, job](HostSink& sk, int64_t need_n, int64_t est, int64_t have) -> Status {
        PinnedBuf nci = pinned_acquire(static_cast<size_t>(est) * 8), nv = pinned_acquire(static_cast<size_t>(est) * 8);
        if (!nci.p || !nv.p) {
            pinned_release(nci);
            pinned_release(nv);
            return fail(MCMI_ENOMEM, "cudaHostAlloc of " + std::to_string(need_n) + " result entries failed");
        }
        if (job) job->pause_copier();
        if (have) {
            parallel_copy(nci.p, sk.col_idx, static_cast<size_t>(have) * 8);
            parallel_copy(nv.p, sk.values, static_cast<size_t>(have) * 8);
        }
        pinned_release(r->ci);
        pinned_release(r->v);
        r->ci = nci;
        r->v = nv;
        sk.col_idx = nci.as<int64_t>();
        sk.values = nv.as<double>();
        sk.capacity = static_cast<int64_t>(std::min(nci.bytes, nv.bytes) / 8);
        if (job) job->resume_copier(sk.col_idx, sk.values);
        return ok();
    };
    if (job) {
        sink.queued = [job](int64_t qlo, int64_t qhi, cudaStream_t copy) {
            cudaEvent_t ev = nullptr;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventRecord(ev, copy) != cudaSuccess) {
                cudaGetLastError();
                if (ev) cudaEventDestroy(ev);
                return;  // not delivered early: mcmi_job_finish reports the shorter prefix
            }
            std::lock_guard<std::mutex> lk(job->mu);
            job->landed.push_back({qlo, qhi, ev});
            job->cv.notify_all();
        };
    }
    // the estimate is refreshed after every chunk (the first rows of a stencil
    // are a boundary and under-represent the rest)
    sink.progress = [&](int64_t done, int64_t nnz_so_far, int64_t total) {
        if (!on_estimate) return;
        on_estimate(done >= total ? nnz_so_far
                                  : static_cast<int64_t>(static_cast<double>(nnz_so_far) * total /
                                                         static_cast<double>(std::max<int64_t>(done, 1)) * 1.08) +
                                        1024);
    };
    mcmi_device_csr dc{};
    mcmi_stats ls{};
    st = build_from_host(e, b, c, lo, hi, &dc, &ls, &sink, ap_host);
    release_engine(e);
    if (st.code) return st;
    r->n = rows;
    r->nnz = ls.nnz;
    r->n_chains = ls.n_chains;
    r->max_len = ls.max_len;
    r->stats = ls;
    return ok();
}

}  // namespace

// The SplitSystem of mcmi_augment_and_split, copied to host memory.
struct mcmi_split_system {
    int64_t n = 0, nnz_bh = 0, nnz_a = 0;
    double a_norm = 0.0;
    std::vector<int64_t> bh_rp, bh_ci, a_rp, a_ci;
    std::vector<double> bh_v, b1, a_v, p_v, s_diag;
};

namespace {

// Stream-ordered device temporaries of one fine-grained call (freed on scope exit).
struct DevTemps {
    cudaStream_t s;
    std::vector<void*> ptrs;
    cudaError_t err = cudaSuccess;
    explicit DevTemps(cudaStream_t st) : s(st) {}
    template <class T>
    T* get(int64_t count) {
        void* p = nullptr;
        if (err == cudaSuccess) err = cudaMallocAsync(&p, static_cast<size_t>(std::max<int64_t>(count, 1)) * sizeof(T), s);
        if (p) ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~DevTemps() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
    }
};

Status check_host_view(const mcmi_csr_view* b) {
    if (!b) return fail(MCMI_EINVAL, "null argument");
    if (b->n < 0) return fail(MCMI_EINVAL, "negative dimension");
    if (b->n > 0 && !b->row_ptr) return fail(MCMI_EINVAL, "null row_ptr");
    const int64_t nnz = b->n > 0 ? b->row_ptr[b->n] : 0;
    if (nnz < 0) return fail(MCMI_EINVAL, "row_ptr[n] is negative");
    if (nnz > 0 && (!b->col_idx || !b->values)) return fail(MCMI_EINVAL, "null col_idx / values");
    return ok();
}

// Stages a host CSR on the engine's stream and validates its row pointer.
Status stage_csr(mcmi_engine* e, const mcmi_csr_view& b, DevTemps& t, mcmi_csr_view* dv) {
    const int64_t n = b.n, nnz = n > 0 ? b.row_ptr[n] : 0;
    cudaStream_t s = e->own;
    auto* rp = t.get<int64_t>(n + 1);
    auto* ci = t.get<int64_t>(nnz);
    auto* v = t.get<double>(nnz);
    MCMI_TRY(t.err, "alloc staging");
    MCMI_TRY(cudaMemcpyAsync(rp, b.row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, s), "H2D");
    if (nnz) {
        MCMI_TRY(cudaMemcpyAsync(ci, b.col_idx, nnz * sizeof(int64_t), cudaMemcpyDefault, s), "H2D");
        MCMI_TRY(cudaMemcpyAsync(v, b.values, nnz * sizeof(double), cudaMemcpyDefault, s), "H2D");
    }
    MCMI_TRY(e->red.ensure(sizeof(Reductions)), "alloc reductions");
    Reductions init{};
    init.offmin_bits = 0x7ff0000000000000ull;
    init.degenerate_row = LLONG_MAX;
    init.bad_col_row = LLONG_MAX;
    init.bad_rowptr_row = LLONG_MAX;
    *e->h_red = init;
    MCMI_TRY(cudaMemcpyAsync(e->red.p, e->h_red, sizeof(Reductions), cudaMemcpyHostToDevice, s), "init reductions");
    MCMI_TRY(launch_validate_row_ptr(rp, n, nnz, e->red.as<Reductions>(), s), "validate row_ptr");
    MCMI_TRY(cudaMemcpyAsync(e->h_red, e->red.p, sizeof(Reductions), cudaMemcpyDeviceToHost, s), "read validation");
    MCMI_TRY(cudaStreamSynchronize(s), "validate row_ptr");
    if (e->h_red->bad_rowptr_row != LLONG_MAX)
        return fail(MCMI_EINVAL,
                    "row_ptr is not a valid CSR row pointer at row " + std::to_string(e->h_red->bad_rowptr_row));
    *dv = mcmi_csr_view{n, rp, ci, v};
    return ok();
}

template <class T>
Status d2h_vec(std::vector<T>& dst, const T* src, int64_t count, cudaStream_t s) {
    dst.resize(static_cast<size_t>(std::max<int64_t>(count, 0)));
    if (count > 0) MCMI_TRY(cudaMemcpyAsync(dst.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    return ok();
}

Status augment_and_split_dev(mcmi_engine* e, const mcmi_csr_view& b, double alpha, int mode,
                             mcmi_split_system* out) {
    if (!(alpha > 0.0)) return fail(MCMI_EINVAL, "alpha must be positive");  // split.cpp:48
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    DevTemps t(s);
    mcmi_csr_view dv{};
    if (Status st = stage_csr(e, b, t, &dv); st.code) return st;
    const int64_t n = b.n;
    SplitExportArgs a{};
    a.n = n;
    a.row_ptr = dv.row_ptr;
    a.col_idx = dv.col_idx;
    a.values = dv.values;
    a.alpha = alpha;
    a.mode = mode;
    a.red = e->red.as<Reductions>();
    a.diag_val = t.get<double>(n);
    a.has_diag = t.get<unsigned char>(n);
    a.bh_cnt = t.get<int>(n);
    a.a_cnt = t.get<int>(n);
    a.b1_diag = t.get<double>(n);
    a.s_diag = t.get<double>(n);
    int64_t* bh_rp = t.get<int64_t>(n + 1);
    int64_t* a_rp = t.get<int64_t>(n + 1);
    a.bh_row_ptr = bh_rp;
    a.a_row_ptr = a_rp;
    MCMI_TRY(t.err, "alloc split");
    MCMI_TRY(e->scan_tmp.ensure(scan_scratch_bytes(std::max<int64_t>(n, 1)) + 64), "alloc scan");
    MCMI_TRY(launch_split_export(a, 0, s), "split kernels");
    MCMI_TRY(cudaMemcpyAsync(e->h_red, e->red.p, sizeof(Reductions), cudaMemcpyDeviceToHost, s), "read split");
    MCMI_TRY(cudaStreamSynchronize(s), "split kernels");
    const Reductions red = *e->h_red;
    if (red.bad_col_row != LLONG_MAX)
        return fail(MCMI_ERANGE, "column index out of range in row " + std::to_string(red.bad_col_row));
    if (red.degenerate_row != LLONG_MAX)  // split.cpp:67-69
        return fail(MCMI_ESPLIT, "degenerate diagonal after augmentation at row " + std::to_string(red.degenerate_row));
    double a_norm;
    std::memcpy(&a_norm, &red.anorm_bits, sizeof(double));
    if (!(a_norm < 1.0))  // split.cpp:94-96
        return fail(MCMI_ESPLIT, "diagonal dominance failure: ||A||inf = " + std::to_string(a_norm));
    MCMI_TRY(scan_rows_exclusive(a.bh_cnt, bh_rp, n, e->scan_tmp.p, s), "scan");
    MCMI_TRY(scan_rows_exclusive(a.a_cnt, a_rp, n, e->scan_tmp.p, s), "scan");
    int64_t tot[2] = {0, 0};
    MCMI_TRY(cudaMemcpyAsync(&tot[0], bh_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaMemcpyAsync(&tot[1], a_rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "scan");
    a.bh_col = t.get<int64_t>(tot[0]);
    a.bh_val = t.get<double>(tot[0]);
    a.a_col = t.get<int64_t>(tot[1]);
    a.a_val = t.get<double>(tot[1]);
    a.p_val = t.get<double>(tot[1]);
    MCMI_TRY(t.err, "alloc split");
    MCMI_TRY(launch_split_export(a, 1, s), "split fill");
    out->n = n;
    out->nnz_bh = tot[0];
    out->nnz_a = tot[1];
    out->a_norm = a_norm;
    Status st;
    for (Status x : {d2h_vec(out->bh_rp, static_cast<const int64_t*>(bh_rp), n + 1, s),
                     d2h_vec(out->bh_ci, static_cast<const int64_t*>(a.bh_col), tot[0], s),
                     d2h_vec(out->bh_v, static_cast<const double*>(a.bh_val), tot[0], s),
                     d2h_vec(out->b1, static_cast<const double*>(a.b1_diag), n, s),
                     d2h_vec(out->s_diag, static_cast<const double*>(a.s_diag), n, s),
                     d2h_vec(out->a_rp, static_cast<const int64_t*>(a_rp), n + 1, s),
                     d2h_vec(out->a_ci, static_cast<const int64_t*>(a.a_col), tot[1], s),
                     d2h_vec(out->a_v, static_cast<const double*>(a.a_val), tot[1], s),
                     d2h_vec(out->p_v, static_cast<const double*>(a.p_val), tot[1], s)})
        if (x.code && !st.code) st = x;
    if (st.code) return st;
    MCMI_TRY(cudaStreamSynchronize(s), "split D2H");
    if (n == 0) out->bh_rp.assign(1, 0), out->a_rp.assign(1, 0);
    return ok();
}

Status drop_small_entries_dev(mcmi_engine* e, const mcmi_csr_view& m, double p, int drop_mode, int64_t* o_rp,
                              int64_t* o_ci, double* o_v, int64_t* o_nnz) {
    if (!(p >= 0.0 && p <= 1.0)) return fail(MCMI_EINVAL, "drop fraction must lie in [0,1]");  // csr.cpp:128-129
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    DevTemps t(s);
    mcmi_csr_view dv{};
    if (Status st = stage_csr(e, m, t, &dv); st.code) return st;
    const int64_t n = m.n, nnz = n > 0 ? m.row_ptr[n] : 0;
    TableBuildArgs ta{};
    ta.n = n;
    ta.row_ptr = dv.row_ptr;
    ta.col_idx = dv.col_idx;
    ta.values = dv.values;
    ta.drop_fraction = p;
    ta.drop_mode = drop_mode;
    ta.red = e->red.as<Reductions>();
    const bool active = p != 0.0 && n > 0;
    if (active && drop_mode == MCMI_DROP_COUNT_QUANTILE) {
        MCMI_TRY(e->keep.ensure(std::max<int64_t>(nnz, 1)), "alloc keep");
        MCMI_TRY(e->cq_tmp.ensure(count_quantile_scratch_bytes(std::max<int64_t>(nnz, 1))), "alloc cq");
        ta.keep = e->keep.as<unsigned char>();
        MCMI_TRY(launch_count_quantile(ta, nnz, 0, e->cq_tmp.p, e->cq_tmp.cap, s), "count-quantile drop");
    }
    int* cnt = t.get<int>(n);
    int64_t* orp = t.get<int64_t>(n + 1);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(e->scan_tmp.ensure(scan_scratch_bytes(std::max<int64_t>(n, 1)) + 64), "alloc scan");
    MCMI_TRY(launch_drop_filter(ta, active, 0, cnt, nullptr, nullptr, nullptr, s), "drop count");
    MCMI_TRY(scan_rows_exclusive(cnt, orp, n, e->scan_tmp.p, s), "scan");
    int64_t tot = 0;
    if (n > 0) MCMI_TRY(cudaMemcpyAsync(&tot, orp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "scan");
    int64_t* oci = t.get<int64_t>(tot);
    double* ov = t.get<double>(tot);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(launch_drop_filter(ta, active, 1, nullptr, orp, oci, ov, s), "drop fill");
    if (n > 0) MCMI_TRY(cudaMemcpyAsync(o_rp, orp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    if (tot) {
        MCMI_TRY(cudaMemcpyAsync(o_ci, oci, tot * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
        MCMI_TRY(cudaMemcpyAsync(o_v, ov, tot * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    }
    MCMI_TRY(cudaStreamSynchronize(s), "D2H");
    if (n == 0) o_rp[0] = 0;
    *o_nnz = tot;
    return ok();
}

// retain_top_k (mc_engine.cpp:124-145) of every row of `m` (rowops.cu).
Status retain_top_k_dev(mcmi_engine* e, const mcmi_csr_view& m, int64_t k, const int64_t* diag_cols, int64_t* o_rp,
                        int64_t* o_ci, double* o_v, int64_t* o_nnz) {
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    DevTemps t(s);
    mcmi_csr_view dv{};
    if (Status st = stage_csr(e, m, t, &dv); st.code) return st;
    const int64_t n = m.n;
    int64_t* d_diag = nullptr;
    if (diag_cols && n > 0) {
        d_diag = t.get<int64_t>(n);
        MCMI_TRY(t.err, "alloc");
        MCMI_TRY(cudaMemcpyAsync(d_diag, diag_cols, n * sizeof(int64_t), cudaMemcpyDefault, s), "H2D");
    }
    int* cnt = t.get<int>(n);
    int64_t* orp = t.get<int64_t>(n + 1);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(e->scan_tmp.ensure(scan_scratch_bytes(std::max<int64_t>(n, 1)) + 64), "alloc scan");
    MCMI_TRY(launch_topk_rows(dv.row_ptr, dv.col_idx, dv.values, n, k, d_diag, 0, cnt, nullptr, nullptr, nullptr, s),
             "top-k count");
    MCMI_TRY(scan_rows_exclusive(cnt, orp, n, e->scan_tmp.p, s), "scan");
    int64_t tot = 0;
    if (n > 0) MCMI_TRY(cudaMemcpyAsync(&tot, orp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "scan");
    int64_t* oci = t.get<int64_t>(tot);
    double* ov = t.get<double>(tot);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(launch_topk_rows(dv.row_ptr, dv.col_idx, dv.values, n, k, d_diag, 1, cnt, orp, oci, ov, s), "top-k");
    if (n > 0) MCMI_TRY(cudaMemcpyAsync(o_rp, orp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    if (tot) {
        MCMI_TRY(cudaMemcpyAsync(o_ci, oci, tot * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
        MCMI_TRY(cudaMemcpyAsync(o_v, ov, tot * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    }
    MCMI_TRY(cudaStreamSynchronize(s), "D2H");
    if (n == 0) o_rp[0] = 0;
    *o_nnz = tot;
    return ok();
}

// scale_columns (mc_engine.cpp:147-149) of every entry of `m` (rowops.cu).
Status scale_columns_dev(mcmi_engine* e, const mcmi_csr_view& m, const double* b1, int64_t b1_len, double* o_v) {
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    DevTemps t(s);
    mcmi_csr_view dv{};
    if (Status st = stage_csr(e, m, t, &dv); st.code) return st;
    const int64_t nnz = m.n > 0 ? m.row_ptr[m.n] : 0;
    if (nnz == 0) return ok();
    double* d_b1 = t.get<double>(b1_len);
    double* d_out = t.get<double>(nnz);
    int* bad = t.get<int>(1);
    MCMI_TRY(t.err, "alloc");
    if (b1_len > 0) MCMI_TRY(cudaMemcpyAsync(d_b1, b1, b1_len * sizeof(double), cudaMemcpyDefault, s), "H2D");
    MCMI_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
    MCMI_TRY(launch_scale_columns(dv.col_idx, dv.values, nnz, d_b1, b1_len, d_out, bad, s), "scale_columns");
    int h_bad = 0;
    MCMI_TRY(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "scale_columns");
    if (h_bad) return fail(MCMI_ERANGE, "column index outside b1_diag");
    MCMI_TRY(cudaMemcpyAsync(o_v, d_out, nnz * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "D2H");
    return ok();
}

Status transition_probabilities_dev(mcmi_engine* e, const mcmi_csr_view& a, int64_t* p_rp, int64_t* p_ci,
                                    double* p_v, int64_t* p_nnz) {
    MCMI_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    cudaStream_t s = e->own;
    DevTemps t(s);
    mcmi_csr_view dv{};
    if (Status st = stage_csr(e, a, t, &dv); st.code) return st;
    const int64_t n = a.n;
    int* cnt = t.get<int>(n);
    int64_t* orp = t.get<int64_t>(n + 1);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(e->scan_tmp.ensure(scan_scratch_bytes(std::max<int64_t>(n, 1)) + 64), "alloc scan");
    MCMI_TRY(launch_transition_probabilities(dv.row_ptr, dv.col_idx, dv.values, n, cnt, nullptr, nullptr, nullptr, 0, s),
             "transition counts");
    MCMI_TRY(scan_rows_exclusive(cnt, orp, n, e->scan_tmp.p, s), "scan");
    int64_t tot = 0;
    MCMI_TRY(cudaMemcpyAsync(&tot, orp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    MCMI_TRY(cudaStreamSynchronize(s), "scan");
    int64_t* oci = t.get<int64_t>(tot);
    double* ov = t.get<double>(tot);
    MCMI_TRY(t.err, "alloc");
    MCMI_TRY(launch_transition_probabilities(dv.row_ptr, dv.col_idx, dv.values, n, nullptr, orp, oci, ov, 1, s),
             "transition fill");
    MCMI_TRY(cudaMemcpyAsync(p_rp, orp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
    if (tot) {
        MCMI_TRY(cudaMemcpyAsync(p_ci, oci, tot * sizeof(int64_t), cudaMemcpyDeviceToHost, s), "D2H");
        MCMI_TRY(cudaMemcpyAsync(p_v, ov, tot * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    }
    MCMI_TRY(cudaStreamSynchronize(s), "D2H");
    if (n == 0) p_rp[0] = 0;
    *p_nnz = tot;
    return ok();
}

}  // namespace

extern "C" {

void mcmi_config_default(mcmi_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->epsilon = 0.0625;
    c->delta = 0.0625;
    c->alpha = 5.0;
    c->mode = MCMI_AUGMENT_SIGN_AWARE;
    c->drop_mode = MCMI_DROP_VALUE_RANGE;
    c->rng_mode = MCMI_RNG_REFERENCE;
}

const char* mcmi_version(void) { return "mcmi 1 sm_100a"; }

int mcmi_engine_create(int device, mcmi_engine** out, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    *out = nullptr;
    auto* e = new mcmi_engine();
    Status st = engine_init(e, device);
    if (st.code) {
        engine_release(e);
        delete e;
        return report(st, err, errlen);
    }
    *out = e;
    return MCMI_OK;
}

void mcmi_engine_destroy(mcmi_engine* e) {
    const mcmi::DeviceGuard device_guard;
    if (!e) return;
    engine_release(e);
    delete e;
}

int mcmi_engine_build(mcmi_engine* e, const mcmi_csr_view* b, const mcmi_config* cfg,
                      int64_t row_begin, int64_t row_end, void* stream, mcmi_device_csr* out,
                      mcmi_stats* stats, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!e || !b || !cfg || !out) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->own;
    return report(engine_build(e, *b, *cfg, row_begin, row_end, s, out, stats), err, errlen);
}

int mcmi_build(const mcmi_csr_view* b, const mcmi_config* cfg, mcmi_result** out, char* err,
               size_t errlen) {
    return mcmi_build_rows(b, cfg, 0, -1, out, err, errlen);
}

int mcmi_build_rows(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin,
                    int64_t row_end, mcmi_result** out, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!out) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    *out = nullptr;
    if (!b || !cfg) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    auto* r = new mcmi_result();
    const Status st = build_host(*b, *cfg, row_begin, row_end, r, nullptr, 0.0);
    if (st.code) {
        delete r;
        return report(st, err, errlen);
    }
    *out = r;
    return MCMI_OK;
}

int mcmi_estimate_rows(const mcmi_csr_view* a, const double* p_values, int64_t row_begin, int64_t row_end,
                       int64_t n_chains, int64_t max_len, double delta, uint64_t seed, int32_t rng_mode, int device,
                       mcmi_result** out, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!out) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    *out = nullptr;
    if (!a || (a->n > 0 && a->row_ptr && a->row_ptr[a->n] > 0 && !p_values))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    mcmi_config c;
    mcmi_config_default(&c);
    c.delta = delta;
    c.master_seed = seed;
    c.rng_mode = rng_mode;
    c.device = device;
    c.n_gpus = 1;
    c.flags = MCMI_FLAG_UNSCALED;
    const ApSource ap{p_values, n_chains, max_len};
    auto* r = new mcmi_result();
    const Status st = build_host(*a, c, row_begin, row_end, r, nullptr, 0.0, &ap);
    if (st.code) {
        delete r;
        return report(st, err, errlen);
    }
    *out = r;
    return MCMI_OK;
}

int mcmi_build_start(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin, int64_t row_end,
                     mcmi_job** job, char* err, size_t errlen) {
    if (!job) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    *job = nullptr;
    if (!b || !cfg) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    auto* j = new mcmi_job();
    j->b = *b;
    j->cfg = *cfg;
    j->lo = row_begin;
    j->hi = row_end;
    try {
        j->copier = std::thread([j] { j->copier_loop(); });
        j->th = std::thread([j] {
            auto* r = new mcmi_result();
            auto publish = [j](int64_t est) {
                std::lock_guard<std::mutex> lk(j->mu);
                j->estimate = j->has_estimate ? std::max(j->estimate, est) : est;  // never lowered
                j->has_estimate = true;
                j->cv.notify_all();
            };
            // a small first chunk (5% of the rows) gives the caller its entry
            // estimate early enough to size its own arrays while the walks run
            const Status st = build_host(j->b, j->cfg, j->lo, j->hi, r, publish, 0.05, nullptr, j);
            {
                std::lock_guard<std::mutex> lk(j->mu);
                j->build_over = true;
                j->cv.notify_all();
            }
            if (j->copier.joinable()) j->copier.join();
            std::lock_guard<std::mutex> lk(j->mu);
            for (auto& rg : j->landed) cudaEventDestroy(rg.ev);
            j->landed.clear();
            if (st.code) {
                delete r;
                r = nullptr;
            } else {
                j->has_estimate = true;
                j->estimate = r->nnz;  // exact once built
            }
            j->code = st.code;
            j->msg = st.msg;
            j->result = r;
            j->done = true;
            j->cv.notify_all();
        });
    } catch (const std::exception& ex) {
        if (j->copier.joinable()) {
            {
                std::lock_guard<std::mutex> lk(j->mu);
                j->build_over = true;
                j->cv.notify_all();
            }
            j->copier.join();
        }
        delete j;
        return report(fail(MCMI_ENOMEM, std::string("cannot start the build thread: ") + ex.what()), err, errlen);
    }
    *job = j;
    return MCMI_OK;
}

int mcmi_job_estimate(mcmi_job* job, int64_t* nnz_estimate) {
    if (!job || !nnz_estimate) return MCMI_EINVAL;
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [&] { return job->has_estimate || job->done; });
    *nnz_estimate = job->has_estimate ? job->estimate : -1;
    return job->done ? job->code : MCMI_OK;
}

int mcmi_job_attach(mcmi_job* job, int64_t* col_idx, double* values, int64_t capacity) {
    if (!job || (capacity > 0 && (!col_idx || !values))) return MCMI_EINVAL;
    std::lock_guard<std::mutex> lk(job->mu);
    if (capacity <= 0) return MCMI_OK;
    if (job->dst_col && (job->dst_col != col_idx || job->dst_val != values)) return MCMI_EINVAL;  // same arrays
    job->dst_col = col_idx;
    job->dst_val = values;
    job->dst_cap = std::max(job->dst_cap, capacity);  // the caller's arrays grow while the build runs
    job->cv.notify_all();
    return MCMI_OK;
}

int mcmi_job_finish(mcmi_job* job, mcmi_result** out, int64_t* delivered, char* err, size_t errlen) {
    if (delivered) *delivered = 0;
    if (!job) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    if (job->th.joinable()) job->th.join();
    if (delivered && job->result) *delivered = std::min(job->delivered, job->result->nnz);
    const Status st{job->code, job->msg};
    if (out) {
        *out = job->result;
    } else if (job->result) {
        delete job->result;
    }
    delete job;
    return report(st, err, errlen);
}

int mcmi_build_into(const mcmi_csr_view* b, const mcmi_config* cfg, int64_t row_begin, int64_t row_end,
                    int64_t* row_ptr, int64_t* col_idx, double* values, int64_t capacity,
                    int64_t* chains_used, int64_t* entries_before, int64_t* nnz, mcmi_stats* stats,
                    char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!b || !cfg || !row_ptr || !nnz || (capacity > 0 && (!col_idx || !values)))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    std::vector<int> devs;
    if (Status st = shard_devices(*cfg, &devs); st.code) return report(st, err, errlen);
    if (devs.size() > 1) {
        // several GPUs: shards are built concurrently, then each GPU copies its
        // shard straight to its global offset (offsets are known only after
        // every shard has its entry count, so the copies do not overlap the walks)
        DeviceParts r;
        Status st = build_parts(*b, *cfg, row_begin, row_end, &r);
        if (st.code) return report(st, err, errlen);
        *nnz = r.nnz;
        if (stats) *stats = r.stats;
        int code = MCMI_OK;
        if (r.nnz > capacity) {
            st = fail(MCMI_ENOMEM, "output capacity " + std::to_string(capacity) + " < nnz " + std::to_string(r.nnz));
        } else {
            code = copy_parts(&r, row_ptr, col_idx, values, chains_used, entries_before);
            if (code) st = fail(code, "device->host copy failed");
        }
        free_parts(&r);
        return report(st, err, errlen);
    }
    mcmi_config c = *cfg;
    c.device = devs[0];
    Status st;
    mcmi_engine* e = acquire_engine(c.device, &st);
    if (!e) return report(st, err, errlen);
    HostSink sink;
    sink.row_ptr = row_ptr;
    sink.col_idx = col_idx;
    sink.values = values;
    sink.capacity = capacity;
    sink.chains_used = chains_used;
    sink.entries_before = entries_before;
    mcmi_device_csr dc{};
    mcmi_stats ls{};
    st = build_from_host(e, *b, c, row_begin, row_end, &dc, &ls, &sink);
    *nnz = ls.nnz;
    if (stats) *stats = ls;
    release_engine(e);
    return report(st, err, errlen);
}

int mcmi_derive_chain_budget(const mcmi_config* cfg, double a_norm, int64_t* n_chains, int64_t* max_len, char* err,
                             size_t errlen) {
    if (!cfg || !n_chains || !max_len) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    return report(chain_budget(*cfg, a_norm, n_chains, max_len), err, errlen);
}

int mcmi_augment_and_split(const mcmi_csr_view* b, double alpha, int32_t mode, int device, mcmi_split_system** out,
                           char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!out) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    *out = nullptr;
    if (Status st = check_host_view(b); st.code) return report(st, err, errlen);
    Status st;
    mcmi_engine* e = acquire_engine(device, &st);
    if (!e) return report(st, err, errlen);
    auto* r = new mcmi_split_system();
    st = augment_and_split_dev(e, *b, alpha, mode, r);
    release_engine(e);
    if (st.code) {
        delete r;
        return report(st, err, errlen);
    }
    *out = r;
    return MCMI_OK;
}

int mcmi_split_sizes(const mcmi_split_system* s, int64_t* n, int64_t* nnz_b_hat, int64_t* nnz_a, double* a_norm) {
    if (!s) return MCMI_EINVAL;
    if (n) *n = s->n;
    if (nnz_b_hat) *nnz_b_hat = s->nnz_bh;
    if (nnz_a) *nnz_a = s->nnz_a;
    if (a_norm) *a_norm = s->a_norm;
    return MCMI_OK;
}

int mcmi_split_copy(const mcmi_split_system* s, int64_t* b_hat_row_ptr, int64_t* b_hat_col_idx, double* b_hat_values,
                    double* b1_diag, int64_t* a_row_ptr, int64_t* a_col_idx, double* a_values, double* p_values,
                    double* s_diag) {
    if (!s) return MCMI_EINVAL;
    auto cp = [](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    cp(b_hat_row_ptr, s->bh_rp.data(), s->bh_rp.size() * sizeof(int64_t));
    cp(b_hat_col_idx, s->bh_ci.data(), s->bh_ci.size() * sizeof(int64_t));
    cp(b_hat_values, s->bh_v.data(), s->bh_v.size() * sizeof(double));
    cp(b1_diag, s->b1.data(), s->b1.size() * sizeof(double));
    cp(a_row_ptr, s->a_rp.data(), s->a_rp.size() * sizeof(int64_t));
    cp(a_col_idx, s->a_ci.data(), s->a_ci.size() * sizeof(int64_t));
    cp(a_values, s->a_v.data(), s->a_v.size() * sizeof(double));
    cp(p_values, s->p_v.data(), s->p_v.size() * sizeof(double));
    cp(s_diag, s->s_diag.data(), s->s_diag.size() * sizeof(double));
    return MCMI_OK;
}

void mcmi_split_free(mcmi_split_system* s) { delete s; }

int mcmi_transition_probabilities(const mcmi_csr_view* a, int device, int64_t* p_row_ptr, int64_t* p_col_idx,
                                  double* p_values, int64_t* p_nnz, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!p_row_ptr || !p_nnz) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    if (Status st = check_host_view(a); st.code) return report(st, err, errlen);
    if (a->n > 0 && a->row_ptr[a->n] > 0 && (!p_col_idx || !p_values))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    Status st;
    mcmi_engine* e = acquire_engine(device, &st);
    if (!e) return report(st, err, errlen);
    st = transition_probabilities_dev(e, *a, p_row_ptr, p_col_idx, p_values, p_nnz);
    release_engine(e);
    return report(st, err, errlen);
}

int mcmi_drop_small_entries(const mcmi_csr_view* m, double p, int32_t drop_mode, int device, int64_t* out_row_ptr,
                            int64_t* out_col_idx, double* out_values, int64_t* out_nnz, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!out_row_ptr || !out_nnz) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    if (Status st = check_host_view(m); st.code) return report(st, err, errlen);
    if (m->n > 0 && m->row_ptr[m->n] > 0 && (!out_col_idx || !out_values))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    Status st;
    mcmi_engine* e = acquire_engine(device, &st);
    if (!e) return report(st, err, errlen);
    st = drop_small_entries_dev(e, *m, p, drop_mode, out_row_ptr, out_col_idx, out_values, out_nnz);
    release_engine(e);
    return report(st, err, errlen);
}

int mcmi_retain_top_k(const mcmi_csr_view* rows, int64_t k, const int64_t* diag_cols, int device,
                      int64_t* out_row_ptr, int64_t* out_col_idx, double* out_values, int64_t* out_nnz, char* err,
                      size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (!out_row_ptr || !out_nnz) return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    if (Status st = check_host_view(rows); st.code) return report(st, err, errlen);
    if (rows->n > 0 && rows->row_ptr[rows->n] > 0 && (!out_col_idx || !out_values))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    Status st;
    mcmi_engine* e = acquire_engine(device, &st);
    if (!e) return report(st, err, errlen);
    st = retain_top_k_dev(e, *rows, k, diag_cols, out_row_ptr, out_col_idx, out_values, out_nnz);
    release_engine(e);
    return report(st, err, errlen);
}

int mcmi_scale_columns(const mcmi_csr_view* rows, const double* b1_diag, int64_t b1_len, int device,
                       double* out_values, char* err, size_t errlen) {
    const mcmi::DeviceGuard device_guard;
    if (Status st = check_host_view(rows); st.code) return report(st, err, errlen);
    if (rows->n > 0 && rows->row_ptr[rows->n] > 0 && (!out_values || !b1_diag))
        return report(fail(MCMI_EINVAL, "null argument"), err, errlen);
    Status st;
    mcmi_engine* e = acquire_engine(device, &st);
    if (!e) return report(st, err, errlen);
    st = scale_columns_dev(e, *rows, b1_diag, b1_len, out_values);
    release_engine(e);
    return report(st, err, errlen);
}

int mcmi_partition_rows(const int64_t* row_ptr, int64_t row_begin, int64_t row_end, int parts, int64_t* edges) {
    if (!row_ptr || !edges || parts < 1 || row_begin < 0 || row_end < row_begin) return MCMI_EINVAL;
    const std::vector<int64_t> e = partition_rows(row_ptr, row_begin, row_end, parts);
    std::copy(e.begin(), e.end(), edges);
    return MCMI_OK;
}

int mcmi_result_sizes(const mcmi_result* r, int64_t* n, int64_t* nnz) {
    if (!r) return MCMI_EINVAL;
    if (n) *n = r->n;
    if (nnz) *nnz = r->nnz;
    return MCMI_OK;
}

int mcmi_result_copy(const mcmi_result* r, int64_t* row_ptr, int64_t* col_idx, double* values,
                     int64_t* chains_used, int64_t* entries_before, int64_t* n_chains,
                     int64_t* max_len) {
    if (!r) return MCMI_EINVAL;
    auto cp = [](void* dst, const PinnedBuf& src, int64_t count) {
        if (dst && src.p && count > 0) parallel_copy(dst, src.p, static_cast<size_t>(count) * 8);
    };
    cp(col_idx, r->ci, r->nnz);
    cp(values, r->v, r->nnz);
    cp(row_ptr, r->rp, r->n + 1);
    cp(chains_used, r->cu, r->n);
    cp(entries_before, r->eb, r->n);
    if (n_chains) *n_chains = r->n_chains;
    if (max_len) *max_len = r->max_len;
    return MCMI_OK;
}

int mcmi_result_copy_range(const mcmi_result* r, int64_t begin, int64_t end, int64_t* col_idx, double* values) {
    if (!r || begin < 0 || end < begin || end > r->nnz) return MCMI_EINVAL;
    if (end == begin) return MCMI_OK;
    const size_t bytes = static_cast<size_t>(end - begin) * 8;
    if (col_idx) parallel_copy(col_idx + begin, r->ci.as<int64_t>() + begin, bytes);
    if (values) parallel_copy(values + begin, r->v.as<double>() + begin, bytes);
    return MCMI_OK;
}

int mcmi_result_view(const mcmi_result* r, const int64_t** row_ptr, const int64_t** col_idx, const double** values,
                     const int64_t** chains_used, const int64_t** entries_before) {
    if (!r) return MCMI_EINVAL;
    if (row_ptr) *row_ptr = r->rp.as<const int64_t>();
    if (col_idx) *col_idx = r->nnz ? r->ci.as<const int64_t>() : nullptr;
    if (values) *values = r->nnz ? r->v.as<const double>() : nullptr;
    if (chains_used) *chains_used = r->cu.as<const int64_t>();
    if (entries_before) *entries_before = r->eb.as<const int64_t>();
    return MCMI_OK;
}

int mcmi_result_stats(const mcmi_result* r, mcmi_stats* stats) {
    if (!r || !stats) return MCMI_EINVAL;
    *stats = r->stats;
    return MCMI_OK;
}

void mcmi_result_free(mcmi_result* r) { delete r; }

int mcmi_host_register(void* ptr, size_t bytes) {
    if (!ptr || !bytes) return MCMI_OK;
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        return MCMI_OK;
    }
    return e == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

int mcmi_host_unregister(void* ptr) {
    if (!ptr) return MCMI_OK;
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) cudaGetLastError();
    return e == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

int mcmi_copy(void* dst, const void* src, size_t bytes, void* stream) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault,
                                          static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? MCMI_OK : MCMI_ECUDA;
}

}  // extern "C"
