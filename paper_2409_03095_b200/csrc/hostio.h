// hostio.h — host-memory plumbing of the host drop-in (mcmi_build*, mcmi_job_*):
// a pool of page-locked buffers that hold host-resident results and staging
// bounce buffers, multi-threaded host copies, and pageable -> device staging.
//
// Why (tools/host_probe.cu on the B200 box, 16 host cores, C2-sized arrays of
// 1.28 GB): D2H into pinned memory 56 GB/s vs 17 GB/s into pageable memory;
// H2D from pageable 11 GB/s vs 56 GB/s pinned; cudaMallocHost of 1.28 GB
// takes 460 ms (so buffers are pooled across builds); a 16-thread copy into
// touched memory runs at ~85 GB/s.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace mcmi {

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Page-locked (portable) host buffer of at least `bytes`, reused from the
// process-wide pool when one is free; p == nullptr if the allocation failed.
PinnedBuf pinned_acquire(size_t bytes);
// Returns the buffer to the pool (the pool frees its largest idle buffers
// beyond a cap); resets `b`.
void pinned_release(PinnedBuf& b);

// memcpy over up to `max_threads` host threads (16 by default, one per >= 8 MB).
void parallel_copy(void* dst, const void* src, size_t bytes, int max_threads = 16);

// true when `p` is page-locked host memory (cudaMallocHost / cudaHostRegister)
// or device memory: a plain cudaMemcpyAsync runs at full speed.
bool is_dma_ready(const void* p);

// Host -> device copies on `s`.  Page-locked sources are queued directly;
// pageable ones go through pinned bounce buffers in ONE pipeline over all
// segments (a host copy of chunk i+1 overlaps the DMA of chunk i, with no
// drain between segments); returns when every bounce DMA has completed.
// tools/stage_probe.cu on the B200 box: pinned H2D alone 56 GB/s, a
// 16-thread host copy alone 70 GB/s; 2 x 64 MB buffers and 16 threads measured
// best inside the C++ drop-in, whose own threads fault its result pages meanwhile.
struct H2DSegment {
    void* dst;
    const void* src;
    size_t bytes;
};
cudaError_t stage_h2d(const H2DSegment* segs, int nseg, cudaStream_t s);
inline cudaError_t stage_h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    const H2DSegment seg{dst, src, bytes};
    return stage_h2d(&seg, 1, s);
}

}  // namespace mcmi
