// hostio.cpp — see hostio.h.
#include "hostio.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace mcmi {
namespace {

std::mutex g_pool_mu;
std::vector<PinnedBuf> g_free;  // idle pooled buffers
constexpr size_t kAlign = size_t{2} << 20;
constexpr size_t kCachedMax = size_t{24} << 30;  // idle bytes kept for reuse

size_t idle_bytes() {
    size_t t = 0;
    for (const PinnedBuf& b : g_free) t += b.bytes;
    return t;
}

}  // namespace

PinnedBuf pinned_acquire(size_t bytes) {
    bytes = std::max<size_t>(bytes, 1);
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        size_t best = g_free.size();
        for (size_t i = 0; i < g_free.size(); ++i)
            // smallest idle buffer that fits, but never a much larger one (a
            // bounce-buffer request must not take a pooled multi-GB result slab)
            if (g_free[i].bytes >= bytes && g_free[i].bytes <= 2 * bytes + kAlign &&
                (best == g_free.size() || g_free[i].bytes < g_free[best].bytes))
                best = i;
        if (best != g_free.size()) {
            PinnedBuf b = g_free[best];
            g_free.erase(g_free.begin() + static_cast<long>(best));
            return b;
        }
    }
    // 1/8 headroom: the next build's entry count may differ a little
    size_t want = bytes + bytes / 8;
    want = (want + kAlign - 1) / kAlign * kAlign;
    PinnedBuf b;
    if (cudaHostAlloc(&b.p, want, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        // release idle pooled memory and retry once
        std::vector<PinnedBuf> drop;
        {
            std::lock_guard<std::mutex> lk(g_pool_mu);
            drop.swap(g_free);
        }
        for (PinnedBuf& d : drop) cudaFreeHost(d.p);
        b.p = nullptr;
        if (cudaHostAlloc(&b.p, want, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return PinnedBuf{};
        }
    }
    b.bytes = want;
    return b;
}

void pinned_release(PinnedBuf& b) {
    if (!b.p) return;
    std::vector<PinnedBuf> drop;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_free.push_back(b);
        while (idle_bytes() > kCachedMax && !g_free.empty()) {
            auto it = std::max_element(g_free.begin(), g_free.end(),
                                       [](const PinnedBuf& x, const PinnedBuf& y) { return x.bytes < y.bytes; });
            drop.push_back(*it);
            g_free.erase(it);
        }
    }
    for (PinnedBuf& d : drop) cudaFreeHost(d.p);
    b = PinnedBuf{};
}

namespace {

// Persistent copy workers (thread start-up would cost ~0.5 ms per 16-way copy).
class CopyPool {
  public:
    struct Job {
        std::atomic<int> left{0};
        std::mutex mu;
        std::condition_variable cv;
    };
    struct Task {
        unsigned char* d;
        const unsigned char* s;
        size_t len;
        Job* job;
    };
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed: workers outlive static teardown
        return *pool;
    }
    void run(std::vector<Task>& tasks) {
        if (tasks.empty()) return;
        Job job;
        job.left = static_cast<int>(tasks.size());
        for (Task& t : tasks) t.job = &job;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (size_t i = 1; i < tasks.size(); ++i) q_.push_back(tasks[i]);
        }
        cv_.notify_all();
        execute(tasks[0]);  // the caller takes the first slice, then helps with its own queue
        for (;;) {
            Task t{};
            {
                std::lock_guard<std::mutex> lk(mu_);
                auto it = std::find_if(q_.begin(), q_.end(), [&](const Task& x) { return x.job == &job; });
                if (it == q_.end()) break;
                t = *it;
                q_.erase(it);
            }
            execute(t);
        }
        std::unique_lock<std::mutex> lk(job.mu);
        job.cv.wait(lk, [&] { return job.left.load() == 0; });
    }
    unsigned workers() const { return static_cast<unsigned>(th_.size()); }

  private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned i = 0; i + 1 < std::min(hw, 16u); ++i) th_.emplace_back([this] { loop(); });
        for (auto& t : th_) t.detach();
    }
    static void execute(const Task& t) {
        std::memcpy(t.d, t.s, t.len);
        if (t.job->left.fetch_sub(1) == 1) {
            std::lock_guard<std::mutex> lk(t.job->mu);
            t.job->cv.notify_all();
        }
    }
    void loop() {
        for (;;) {
            Task t{};
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return !q_.empty(); });
                t = q_.front();
                q_.pop_front();
            }
            execute(t);
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Task> q_;
    std::vector<std::thread> th_;
};

}  // namespace

void parallel_copy(void* dst, const void* src, size_t bytes, int max_threads) {
    if (!bytes || dst == src) return;
    const size_t per = size_t{8} << 20;
    CopyPool& pool = CopyPool::get();
    const size_t t = std::min<size_t>({pool.workers() + 1, (bytes + per - 1) / per,
                                       static_cast<size_t>(std::max(1, max_threads))});
    if (t <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    auto* d = static_cast<unsigned char*>(dst);
    const auto* s = static_cast<const unsigned char*>(src);
    // 4 KB-aligned slices so no two threads fault the same page
    const size_t slice = ((bytes + t - 1) / t + 4095) / 4096 * 4096;
    std::vector<CopyPool::Task> tasks;
    for (size_t a = 0; a < bytes; a += slice) tasks.push_back({d + a, s + a, std::min(slice, bytes - a), nullptr});
    pool.run(tasks);
}

bool is_dma_ready(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaError_t stage_h2d(const H2DSegment* segs, int nseg, cudaStream_t s) {
    constexpr int kB = 2;                        // bounce buffers
    constexpr size_t kChunk = size_t{64} << 20;  // per host copy / DMA
    constexpr int kThreads = 16;  // the caller's own threads also fault its result pages meanwhile
    cudaError_t e = cudaSuccess;
    bool any_pageable = false;
    for (int i = 0; i < nseg && e == cudaSuccess; ++i) {
        if (!segs[i].bytes) continue;
        if (segs[i].bytes <= (size_t{4} << 20) || is_dma_ready(segs[i].src))
            e = cudaMemcpyAsync(segs[i].dst, segs[i].src, segs[i].bytes, cudaMemcpyDefault, s);
        else
            any_pageable = true;
    }
    if (e != cudaSuccess || !any_pageable) return e;
    PinnedBuf bb[kB];
    bool have = true;
    for (auto& x : bb) have = have && (x = pinned_acquire(kChunk)).p != nullptr;
    cudaEvent_t ev[kB] = {};
    for (int i = 0; i < kB && have && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    bool used[kB] = {};
    int k = 0;
    for (int i = 0; i < nseg && e == cudaSuccess; ++i) {
        const H2DSegment& g = segs[i];
        if (!g.bytes || g.bytes <= (size_t{4} << 20) || is_dma_ready(g.src)) continue;
        if (!have) {  // no pinned memory: the driver's own (slower) pageable path
            e = cudaMemcpyAsync(g.dst, g.src, g.bytes, cudaMemcpyDefault, s);
            continue;
        }
        for (size_t off = 0; off < g.bytes && e == cudaSuccess; off += kChunk, k = (k + 1) % kB) {
            const size_t len = std::min(kChunk, g.bytes - off);
            if (used[k]) e = cudaEventSynchronize(ev[k]);  // its previous DMA is done
            if (e != cudaSuccess) break;
            parallel_copy(bb[k].p, static_cast<const unsigned char*>(g.src) + off, len, kThreads);
            e = cudaMemcpyAsync(static_cast<unsigned char*>(g.dst) + off, bb[k].p, len, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaEventRecord(ev[k], s);
            used[k] = true;
        }
    }
    for (int j = 0; j < kB; ++j)
        if (used[j]) {
            const cudaError_t w = cudaEventSynchronize(ev[j]);
            if (e == cudaSuccess) e = w;
        }
    for (auto& x : ev)
        if (x) cudaEventDestroy(x);
    for (auto& x : bb) pinned_release(x);
    return e;
}

}  // namespace mcmi
