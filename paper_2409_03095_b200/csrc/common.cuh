// common.cuh — shared device helpers for the B200 MCMCMI build.
//
// Compiled with -fmad=false: every f64 expression on the parity path must
// round exactly like the reference's x86-64 SSE2 build (no FMA contraction,
// proj/CMakeLists.txt has no -march).  IEEE +, *, / and fabs are correctly
// rounded on sm_100a, so sequential sums in the same order give the same bits.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mcmi {

constexpr unsigned FULL_MASK = 0xffffffffu;
constexpr int EMPTY_KEY = -1;

// Philox4x32-10 (Salmon et al. SC'11), identical to RngStream::philox
// (/root/reference/proj/include/mcspai/rng.hpp:44-67): ctr = 4 u32 words,
// key = 2 u32 words, 10 rounds with the Random123 multipliers / Weyl steps.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// The same with the 10 round keys precomputed (rk[2r], rk[2r+1] = key + r *
// Weyl steps): passed as kernel parameters they become constant-bank operands
// of the XORs, so a call is 20 IMAD.WIDE + 20 LOP3 with no key updates.
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t* rk) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ rk[2 * round], lo1, hi0 ^ c.w ^ rk[2 * round + 1], lo0);
    }
    return c;
}

// RngStream::next_double (rng.hpp:32-41): lo word drawn first, 53 bits.
__device__ __forceinline__ double u32pair_to_double(uint32_t lo, uint32_t hi) {
    const unsigned long long u = (static_cast<unsigned long long>(hi) << 32) | lo;
    return static_cast<double>(u >> 11) * 0x1.0p-53;
}

// Non-negative doubles order like their bit patterns: lets atomicMax/Min on
// u64 implement exact max/min reductions (order-independent, so bit-exact).
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
    atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(unsigned long long* p, double v) {
    atomicMin(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

}  // namespace mcmi
