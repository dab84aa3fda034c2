// walk.cu — subsystems (2) random walks and (3) per-row accumulate / top-k /
// scale / prune, fused in one persistent warp-per-row kernel.
//
// Reference: estimate_row_impl (mc_engine.cpp:80-113), sample_transition
// (:64-78), retain_top_k (:124-145), scale_columns (:147-149), the zero prune
// (:174-176) and RowMeta (:169).
//
// Scheduling: one warp owns one row at a time (rows claimed in index order
// from a global cursor, so concurrently walked rows are neighbours and their
// transition records stay L1/L2-resident).  The 32 lanes run 32 chains of the
// row concurrently ("batch"), so the dependent gathers of 32 walks overlap.
//
// RNG keying (WalkArgs::rng_mode):
//   MCMI_RNG_REFERENCE: RngStream(seed, row) with draws numbered across
//     chains (rng.hpp:17-74).  Chain c starts at draw D_c = D_{c-1} + k(D_{c-1}),
//     where k(d) = draws consumed by a walk whose first draw is d — the same
//     function for every chain of the row.  Lane j speculatively walks from
//     D + j*ell; the lanes on the orbit of D (found by pointer doubling over
//     next(j) = j + k_j/ell) are exactly the reference's chains, the rest are
//     discarded.  ell adapts to the observed draws per chain, so a row whose
//     chains all draw the same number of times (the common case) wastes nothing.
//   MCMI_RNG_KEYED: u(row, chain, step) = double #(step&1) of
//     Philox({step>>1, chain, row lo, row hi}, seed); every lane is a chain.
//
// Accumulation order: the reference adds deposits to acc[col] in (chain, step)
// order (RowWorkspace::deposit, mc_engine.cpp:45-51).  Floating-point addition
// is not associative, so each batch logs its deposits [lane][step] in shared
// memory and folds them chain-major: per 32-entry chunk, __match_any_sync
// groups equal columns and the group leader adds its peers in lane order.  The
// per-column sums are therefore bit-identical to the reference's.
//
// Accumulator: an open-addressing hash (int32 column -> f64 sum) per warp in
// shared memory, capacity `cap`; a row that touches more than cap_limit
// columns is abandoned and re-run by the host on a larger tier.
//
// The fold of the other columns is a shuffle chain: lane of group rank i adds
// its weight to its predecessor's running sum in round i.
//
// Finalize (per row, in shared memory): compact the hash, bitonic-sort by
// column, multiply by 1/chains_run, rank for retain_top_k (diag first, |v|
// desc, col asc), divide by b1_diag[col], prune exact zeros off the diagonal,
// write the row to its staging slot.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace mcmi {

constexpr int kDefaultMinBlocks = 6;

namespace {

__host__ __device__ inline int round32(int x) { return (x + 31) & ~31; }

struct WarpSmem {
    double* vals;   // [cap]
    double* log_w;  // [logn]
    int* keys;      // [cap]
    int* log_col;   // [logn]
};

__device__ __forceinline__ WarpSmem carve(unsigned char* base, int cap, int logn) {
    WarpSmem s;
    s.vals = reinterpret_cast<double*>(base);
    s.log_w = s.vals + cap;
    s.keys = reinterpret_cast<int*>(s.log_w + logn);
    s.log_col = s.keys + cap;
    return s;
}

// 256-bit read-only global load (LDG.E.ENL2.256 on sm_100a): a whole 32-byte
// state record in one instruction.
__device__ __forceinline__ void ldg256(const void* p, uint4& lo, uint4& hi) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z),
                   "=r"(hi.w)
                 : "l"(p));
}

// Two consecutive 16-byte {cum, ratio} entries from a 32-byte-aligned address
// in one load.
__device__ __forceinline__ void ldg_pair(const double2* p, double2& a, double2& b) {
    uint4 lo, hi;
    ldg256(p, lo, hi);
    a = make_double2(__hiloint2double(static_cast<int>(lo.y), static_cast<int>(lo.x)),
                     __hiloint2double(static_cast<int>(lo.w), static_cast<int>(lo.z)));
    b = make_double2(__hiloint2double(static_cast<int>(hi.y), static_cast<int>(hi.x)),
                     __hiloint2double(static_cast<int>(hi.w), static_cast<int>(hi.z)));
}

// Insert-or-find; returns the slot or -1 if the table is full.  The key's home
// slot h is probed first (one 4-byte load: most lookups end there, hit or
// empty); past an occupied home slot the probe continues over 4-slot buckets
// starting at h's bucket, one 16-byte load per bucket, slots in order.  A key
// therefore sits in the first slot of that sequence that was empty when it was
// inserted (no deletions while a row is open): an empty home slot or a bucket
// holding an empty slot ends an unsuccessful search.  Concurrent inserts of
// distinct keys (one leader per column in a fold chunk) race only through the
// CAS; the loser re-reads.
template <bool GL>
__device__ __forceinline__ int hash_slot(int* keys, unsigned mask, int shift, int col,
                                         int& n_new) {
    const unsigned h = (static_cast<unsigned>(col) * 0x9E3779B1u) >> shift;
    volatile int* vk = keys;
    const int kh = vk[h];
    if (kh == col) return static_cast<int>(h);
    if (kh == EMPTY_KEY) {
        const int old = atomicCAS(&keys[h], EMPTY_KEY, col);
        if (old == EMPTY_KEY) {
            ++n_new;
            return static_cast<int>(h);
        }
        if (old == col) return static_cast<int>(h);
    }
    unsigned b = h & ~3u;
    for (unsigned visited = 0; visited <= mask;) {
        int4 k4;
        if (GL)
            asm volatile("ld.volatile.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(k4.x), "=r"(k4.y), "=r"(k4.z), "=r"(k4.w)
                         : "l"(keys + b));
        else
            asm volatile("ld.volatile.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(k4.x), "=r"(k4.y), "=r"(k4.z), "=r"(k4.w)
                         : "r"(static_cast<unsigned>(__cvta_generic_to_shared(keys + b))));
        if (k4.x == col) return static_cast<int>(b);
        if (k4.y == col) return static_cast<int>(b + 1);
        if (k4.z == col) return static_cast<int>(b + 2);
        if (k4.w == col) return static_cast<int>(b + 3);
        const int e = k4.x == EMPTY_KEY ? 0 : k4.y == EMPTY_KEY ? 1 : k4.z == EMPTY_KEY ? 2 : k4.w == EMPTY_KEY ? 3 : 4;
        if (e < 4) {
            const int old = atomicCAS(&keys[b + e], EMPTY_KEY, col);
            if (old == EMPTY_KEY) {
                ++n_new;
                return static_cast<int>(b + e);
            }
            continue;  // another leader took the slot: re-read the bucket
        }
        b = (b + 4) & mask;
        visited += 4;
    }
    return -1;
}

// acc += 1.0, k times, with the rounding of k sequential additions.  For
// 1 <= acc < 2^53, every sum that stays below the next power of two 2^(e+1) is
// an exactly representable multiple of ulp(acc), so those additions collapse
// into one exact addition; the addition that crosses 2^(e+1) is performed on
// its own (it may round).  A run therefore costs O(binade crossings), not O(k).
// Out of line: taken a few times per row (the row start, two-binade runs), and
// inlined the compiler if-converts part of it into the fast path.
__device__ __noinline__ double add_ones_slow(double acc, int k) {
    while (k > 0) {
        if (!(acc >= 1.0 && acc < 0x1.0p53)) {  // acc == 0 (row start) or out of range
            acc += 1.0;
            --k;
            continue;
        }
        const double top = __longlong_as_double((__double_as_longlong(acc) & 0x7ff0000000000000ll) +
                                                0x0010000000000000ll);  // 2^(e+1)
        const double room = top - acc;  // exact: acc and top share the ulp grid of acc
        // additions that keep the sum below top: i < room
        const double fit = ceil(room) - 1.0;
        const int j = fit < static_cast<double>(k) ? static_cast<int>(fit) : k;
        if (j > 0) {
            acc += static_cast<double>(j);  // exact
            k -= j;
        }
        if (k > 0) {  // the crossing addition, rounded like the reference's
            acc += 1.0;
            --k;
        }
    }
    return acc;
}

// The same in one addition whenever 1 <= acc < 2^50 and
// acc + k stays below 2^(e+2) (at most one binade crossing).  Proof: with
// u = ulp(acc), the k sequential additions are exact until the one that
// crosses 2^(e+1); that one rounds X + 1 to the 2u grid (ties to even), and
// the remaining m additions are exact again.  A single rounding of acc + k =
// (X + 1) + m gives the same value because m is a multiple of 2u that is an
// EVEN multiple (m * 2^(51-e), e <= 50), so shifting by m preserves both the
// nearest 2u-grid point and, for a tie, its parity.  Everything else (acc < 1,
// two crossings, acc >= 2^50) takes the exact loop.
__device__ __forceinline__ double add_ones(double acc, int k) {
    const int hi = __double2hiint(acc);
    const double top2 = __hiloint2double((hi & 0x7ff00000) + 0x00200000, 0);  // 2^(e+2)
    const double t = acc + static_cast<double>(k);
    // 1 <= acc < 2^50 (sign bit clear): one unsigned range test on the high word
    if (static_cast<unsigned>(hi - 0x3ff00000) < 0x03200000u && t < top2) return t;
    if (acc == 0.0) return static_cast<double>(k);  // a row's start: 0 + 1 + ... + 1 = k exactly
    return add_ones_slow(acc, k);
}

// Keeps the lowest `keep` set bits of mask (keep >= 0).
__device__ __forceinline__ unsigned lowest_bits(unsigned mask, int keep) {
    if (__popc(mask) <= keep) return mask;
    if (keep <= 0) return 0u;
    // position of the keep-th set bit by binary search on prefix popcounts
    int lo = 0, hi = 32;  // answer in [lo, hi): smallest p with popc(mask & ((2<<p)-1)) >= keep
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        const unsigned pre = mid >= 32 ? mask : (mask & ((1u << mid) - 1u));
        if (__popc(pre) >= keep) hi = mid;
        else lo = mid;
    }
    return hi >= 32 ? mask : (mask & ((1u << hi) - 1u));
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

// retain_top_k ordering (mc_engine.cpp:131-139): does entry j precede entry i?
__device__ __forceinline__ bool topk_before(int cj, double vj, int ci, double vi, int diag) {
    const bool dj = cj == diag, di = ci == diag;
    if (dj != di) return dj;
    const double mj = fabs(vj), mi = fabs(vi);
    if (mj != mi) return mj > mi;
    return cj < ci;
}

__device__ __forceinline__ unsigned long long topk_key(int c, double v, int diag) {
    return c == diag ? ~0ull : static_cast<unsigned long long>(__double_as_longlong(fabs(v)));
}

// Warp-cooperative selection of the first k entries of [0, s) in retain_top_k
// order (mc_engine.cpp:131-139: diagonal first, |v| desc, column asc) by a
// radix select over the 64-bit key (8 passes) and, for ties at the threshold,
// over the column (4 passes).  Entry i is kept iff key > T || (key == T &&
// col <= Tc).  hist: 256 scratch words.  O(s) instead of the O(s^2) ranking.
// After the first pass that leaves fewer than s/2 entries in play (those whose
// leading bytes equal the threshold's; values of a row usually share the top
// byte, so typically after the second) they are copied to [s, s + cnt) when at
// most `spare` fit there, and the later passes read only those (wide rows: 4
// passes over the row instead of 9);
// `copied` returns cnt (0 if not copied): those slots must be emptied again.
__device__ void radix_topk(int* keys, double* vals, int s, int k, int diag, unsigned* hist, int spare,
                           unsigned long long& T, int& Tc, int& copied) {
    const int lane = static_cast<int>(threadIdx.x & 31);
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned long long prefix = 0, mask = 0;
    unsigned need = static_cast<unsigned>(k);
    unsigned eq = 0;  // entries matching the full prefix after the last pass
    const int* lk = keys;  // the entries scanned by the passes
    const double* lv = vals;
    int ln = s;
    copied = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int b = lane; b < 256; b += 32) hist[b] = 0;
        __syncwarp();
        // 4 entries per lane in flight: on the global tiers these passes stream
        // MBs per row from HBM, latency-bound at one load pair per iteration
        for (int i0 = lane; i0 < ln; i0 += 128) {
            int kk[4];
            double vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + 32 * u;
                kk[u] = i < ln ? lk[i] : diag;
                vv[u] = i < ln ? lv[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const unsigned long long key = topk_key(kk[u], vv[u], diag);
                if (i0 + 32 * u < ln && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
            }
        }
        __syncwarp();
        unsigned c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // lane owns digits 255-8l .. 248-8l (descending)
            c[j] = hist[255 - 8 * lane - j];
            tot += c[j];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned nb = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += nb;
        }
        const unsigned excl = incl - tot;
        const unsigned owner = __ballot_sync(FULL_MASK, excl < need && need <= incl);
        const int src = __ffs(owner) - 1;
        int d = 0;
        unsigned above = 0, cnt = 0;
        if (lane == src) {
            unsigned cum = excl;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (cum + c[j] >= need) {
                    d = 255 - 8 * lane - j;
                    above = cum;
                    cnt = c[j];
                    break;
                }
                cum += c[j];
            }
        }
        d = __shfl_sync(FULL_MASK, d, src);
        above = __shfl_sync(FULL_MASK, above, src);
        eq = __shfl_sync(FULL_MASK, cnt, src);
        need -= above;
        prefix |= static_cast<unsigned long long>(d) << shift;
        mask |= 0xffull << shift;
        __syncwarp();
        if (ln == s && shift > 0 && eq <= static_cast<unsigned>(spare) && eq < static_cast<unsigned>(s) / 2) {
            int o = 0;
            for (int g0 = 0; g0 < s; g0 += 128) {
                int kk[4];
                double vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = g0 + 32 * u + lane;
                    kk[u] = i < s ? keys[i] : diag;
                    vv[u] = i < s ? vals[i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool in = g0 + 32 * u + lane < s && (topk_key(kk[u], vv[u], diag) & mask) == prefix;
                    const unsigned bal = __ballot_sync(FULL_MASK, in);
                    if (in) {
                        keys[s + o + __popc(bal & lt_mask)] = kk[u];
                        vals[s + o + __popc(bal & lt_mask)] = vv[u];
                    }
                    o += __popc(bal);
                }
            }
            __syncwarp();
            lk = keys + s;
            lv = vals + s;
            ln = o;
            copied = o;
        }
    }
    T = prefix;
    Tc = INT_MAX;
    if (eq > need) {  // keep the `need` smallest columns among the ties
        unsigned cprefix = 0, cmask = 0;
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int b = lane; b < 256; b += 32) hist[b] = 0;
            __syncwarp();
            for (int i = lane; i < ln; i += 32) {
                const unsigned col = static_cast<unsigned>(lk[i]);
                if (topk_key(lk[i], lv[i], diag) == T && (col & cmask) == cprefix)
                    atomicAdd(&hist[(col >> shift) & 255u], 1u);
            }
            __syncwarp();
            unsigned c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // ascending digits 8l .. 8l+7
                c[j] = hist[8 * lane + j];
                tot += c[j];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned nb = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane >= o) incl += nb;
            }
            const unsigned excl = incl - tot;
            const unsigned owner = __ballot_sync(FULL_MASK, excl < need && need <= incl);
            const int src = __ffs(owner) - 1;
            int d = 0;
            unsigned below = 0;
            if (lane == src) {
                unsigned cum = excl;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (cum + c[j] >= need) {
                        d = 8 * lane + j;
                        below = cum;
                        break;
                    }
                    cum += c[j];
                }
            }
            d = __shfl_sync(FULL_MASK, d, src);
            below = __shfl_sync(FULL_MASK, below, src);
            need -= below;
            cprefix |= static_cast<unsigned>(d) << shift;
            cmask |= 0xffu << shift;
            __syncwarp();
        }
        Tc = static_cast<int>(cprefix);
    }
}

// Bitonic sort of (keys, vals)[0, P) by key, P a power of two >= 64.
__device__ void warp_bitonic(int* keys, double* vals, int P) {
    const int lane = static_cast<int>(threadIdx.x & 31);
    for (int kb = 2; kb <= P; kb <<= 1) {
        for (int jb = kb >> 1; jb > 0; jb >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ jb;
                if (ixj > i) {
                    const int ka = keys[i], kc = keys[ixj];
                    const bool up = (i & kb) == 0;
                    if ((ka > kc) == up) {
                        const double va = vals[i];
                        keys[i] = kc;
                        keys[ixj] = ka;
                        vals[i] = vals[ixj];
                        vals[ixj] = va;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Rank sort of (keys, vals)[0, s), s <= 32*E, distinct keys: lane l holds
// entries l, l+32, ...; each entry's destination is the number of smaller
// keys, counted against a broadcast read of every key (s reads per lane, no
// barriers), then everything is scattered at once.
template <int E>
__device__ __forceinline__ void warp_rank_sort(int* keys, double* vals, int s) {
    const int lane = static_cast<int>(threadIdx.x & 31);
    int k[E], r[E];
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        k[e] = i < s ? keys[i] : INT_MAX;
        v[e] = i < s ? vals[i] : 0.0;
        r[e] = 0;
    }
    int j = 0;
    for (; j + 4 <= s; j += 4) {
        const int4 q = *reinterpret_cast<const int4*>(keys + j);
#pragma unroll
        for (int e = 0; e < E; ++e) r[e] += (q.x < k[e]) + (q.y < k[e]) + (q.z < k[e]) + (q.w < k[e]);
    }
    for (; j < s; ++j) {
        const int q = keys[j];
#pragma unroll
        for (int e = 0; e < E; ++e) r[e] += q < k[e];
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (lane + 32 * e < s) {
            keys[r[e]] = k[e];
            vals[r[e]] = v[e];
        }
    __syncwarp();
}

// Sorts (keys, vals)[0, s) by column: rank sorts for s <= 128 (register rank
// sort for s <= 32; 2, 3 or 4 entries per lane up to 64 / 96 / 128), bitonic
// otherwise (pads [s, P) with INT_MAX); returns the
// padded length touched.
__device__ int sort_by_column(int* keys, double* vals, int s) {
    const int lane = static_cast<int>(threadIdx.x & 31);
    if (s <= 32) {
        // columns are distinct: an entry's position is the number of smaller columns
        const int kk = lane < s ? keys[lane] : INT_MAX;
        const double vv = lane < s ? vals[lane] : 0.0;
        int pos = 0;
#pragma unroll 4
        for (int j = 0; j < s; ++j) pos += __shfl_sync(FULL_MASK, kk, j) < kk;
        __syncwarp();
        if (lane < s) {
            keys[pos] = kk;
            vals[pos] = vv;
        }
        __syncwarp();
        return s;
    }
    if (s <= 64) {
        warp_rank_sort<2>(keys, vals, s);
        return s;
    }
    if (s <= 96) {
        warp_rank_sort<3>(keys, vals, s);
        return s;
    }
    if (s <= 128) {
        warp_rank_sort<4>(keys, vals, s);
        return s;
    }
    int P = 64;
    while (P < s) P <<= 1;
    for (int i = s + lane; i < P; i += 32) {
        keys[i] = INT_MAX;
        vals[i] = 0.0;
    }
    __syncwarp();
    warp_bitonic(keys, vals, P);
    return P;
}

constexpr int kRankTopkMax = 256;  // above this row length retain_top_k uses radix_topk

// Neighbourhood slot tables (NB variant, L = 2 with the 32/64/256-slot tiers): at row
// start the warp inserts r's columns and its neighbours' columns into the hash
// once and keeps T1[i] = slot of r's i-th column, T2[off[i] + j] = slot of the
// j-th column of r's i-th neighbour.  A step then logs a slot instead of a
// column (equal slots <=> equal columns, so the (chain, step) fold order is
// unchanged), the fold needs no hash probe, and the last step needs no column
// load.  A touched-slot mask keeps the emitted set = the visited columns.
// Rows whose neighbourhood exceeds the tables or the tier run the plain path.
constexpr int kNbDeg = 32;    // max deg(r)
constexpr int kNbT2 = 704;    // max sum of the neighbours' degrees
constexpr int kNbBytes = 32 + 2 * kNbDeg + kNbDeg + kNbT2;  // mask[8] u32, off[32] u16, T1[32] u8, T2 u8

// Split fold (L = 2 kernels without NB tables, rows flagged by k_tri_free):
// no triangle through r, so a step-0 deposit lands only on a neighbour c_k of
// r, always with the value ratio_k = a/p of transition k (mc_engine.cpp:94),
// and no step-1 deposit lands there.  Column c_k's ordered sum is therefore
// m_k sequential additions of ratio_k, m_k = the chains whose first step took
// transition k: the batches only count them (per-warp counters), the fold of
// the log covers the step-1 deposits alone (one 32-entry chunk per batch
// instead of two), and c_k's sums are formed once per row.  Bit-identical.
constexpr int kTfBytes = 32 * 4;  // per-warp m_k counters (deg(r) <= 16)

// L = 2 deposit-log swizzle: deposit (chain j, step t) of a 32-chain batch sits
// at t*32 + (j ^ 16t) in log_col and t*32 + (j ^ 8t) in log_w, so both the
// walk's writes (one step, all chains) and the fold's chain-major reads (16
// chains x 2 steps per 32-entry chunk) are bank-conflict free: the int reads
// cover banks 0-31 once, and each half-warp's 8-byte reads cover them once.
__device__ __forceinline__ int lf2_col_at(int t, int j) { return t * 32 + (j ^ (t << 4)); }
__device__ __forceinline__ int lf2_w_at(int t, int j) { return t * 32 + (j ^ (t << 3)); }
template <int LF, bool NB>
__host__ __device__ constexpr bool split_fold_kernel() {
    return LF == 2 && !NB;
}

template <int MODE, int MINB, bool GL, bool DEG, int LF = 0, int CAPC = 0, bool NB = false>
__global__ void __launch_bounds__(256, MINB) k_walk(const WalkArgs a) {
    static_assert(!NB || (LF == 2 && CAPC >= 32 && CAPC <= 256 && !GL), "NB: L = 2 kernel, shared tiers");
    // LF > 0: a launch with max_len == log_stride == LF and 32-lane batches:
    // the step loop (unrolled, no length or log-capacity tests) and the fold's
    // position arithmetic are compile-time.
    // MODE 0: reference stream with 32-bit draw positions (N*L < 2^32, every
    // practical budget); MODE 2: the same with 64-bit positions; MODE 1: keyed.
    constexpr bool IS_REF = MODE != 1;
    using PosT = typename std::conditional<MODE == 2, unsigned long long, unsigned>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = static_cast<int>(threadIdx.x & 31);
    const int warp = static_cast<int>(threadIdx.x >> 5);
    const int cap = CAPC ? CAPC : a.cap;  // CAPC: compile-time hash capacity (tiers 32, 64, 256)
    const int S = LF ? LF : a.log_stride;       // step deposits per chain (max_len)
    const int B = LF ? 32 : a.lanes;            // chains per batch
    const int logn = LF ? round32(32 * LF) : a.log_n;  // round32(B * S), host-computed (kernel parameter)
    constexpr bool kTF = split_fold_kernel<LF, NB>();
    // Aligned 32-byte pair loads in the neighbourhood-table kernels (C2 at
    // eps = 0.01, where the L1 data pipe binds: -1.2% reference stream, -2.4%
    // keyed); the other kernels keep two 16-byte loads (C3 +4%, C4 +4% with
    // the aligned form: more spills).  Loading the pair's two columns with it
    // (one 8-byte load) measured no better.
#ifdef MCMI_PAIR_ALL
    constexpr bool kAlignedPair = true;
#else
    constexpr bool kAlignedPair = NB;
#endif
    const size_t per_warp = (LF && CAPC) ? static_cast<size_t>(CAPC + logn) * 12 + (NB ? kNbBytes : 0) +
                                               (kTF ? kTfBytes : 0)
                                         : static_cast<size_t>(a.warp_bytes) + (kTF ? kTfBytes : 0);
    // GL: per-warp accumulator + log in global scratch (large rows / long walks)
    unsigned char* wbase = GL ? a.gscratch + per_warp * (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp)
                              : smem_raw + per_warp * warp;
    const WarpSmem sm = carve(wbase, cap, logn);
    // NB tables after the log (per_warp - kNbBytes)
    unsigned* const nb_mask = NB ? reinterpret_cast<unsigned*>(wbase + (per_warp - kNbBytes)) : nullptr;
    unsigned short* const nb_off = NB ? reinterpret_cast<unsigned short*>(nb_mask + 8) : nullptr;
    unsigned char* const nb_t1 = NB ? reinterpret_cast<unsigned char*>(nb_off + kNbDeg) : nullptr;
    unsigned char* const nb_t2 = NB ? nb_t1 + kNbDeg : nullptr;
    // split-fold counters m_k after the log (per_warp - kTfBytes)
    int* const tf_cnt = kTF ? reinterpret_cast<int*>(wbase + (per_warp - kTfBytes)) : nullptr;
    const unsigned cap_mask = static_cast<unsigned>(cap - 1);
    const int shift = CAPC ? 32 - (31 - __clz(CAPC)) : a.hash_shift;  // 32 - log2(cap)
    const unsigned lt_mask = (1u << lane) - 1u;
    const int s_shift = LF ? (LF == 1 ? 0 : LF == 2 ? 1 : LF == 4 ? 2 : LF == 8 ? 3 : -1) : a.log_shift;  // log2(S), or -1

    const uint4* __restrict__ rec = a.t.rec;
    const double2* __restrict__ ent = a.t.ent;
    const int* __restrict__ tcol = a.t.col;
    // host guarantees 1 <= N < 2^31 and L < 2^31 (engine.cu), so 32-bit loop state
    const int N = static_cast<int>(a.n_chains);
    const int L = LF ? LF : static_cast<int>(a.max_len);

    unsigned long long tot_steps = 0, tot_deg = 0;

    // the accumulator starts empty; finalize restores it to empty after each row
    for (int i = lane; i < cap; i += 32) {
        sm.keys[i] = EMPTY_KEY;
        sm.vals[i] = 0.0;
    }
    __syncwarp();

    // Rows are claimed R = claim_rows consecutive work items at a time (a warp
    // walks neighbouring rows back to back, so their shared 2-hop records are
    // still in its SM's L1), one claim ahead, so the cursor atomic's round trip
    // overlaps the current rows' walks.
    const int R = a.claim_rows;
    int claimed = 0;
    if (lane == 0) claimed = static_cast<int>(atomicAdd(&a.counters[0], static_cast<unsigned long long>(R)));
    int cur = 0, cur_end = 0;
    for (;;) {
        if (cur >= cur_end) {
            cur = __shfl_sync(FULL_MASK, claimed, 0);
            cur_end = cur + R;
            if (cur >= a.n_work) break;
            if (lane == 0) claimed = static_cast<int>(atomicAdd(&a.counters[0], static_cast<unsigned long long>(R)));
        }
        const int wi = cur++;
        if (wi >= a.n_work) {
            cur = cur_end;
            continue;
        }
        const int row = a.row_list ? a.row_list[wi] : static_cast<int>(a.row_begin + a.work_offset) + wi;
        const int rowc = static_cast<int>(row);

        // the diagonal column's slot; its sum lives in a register (acc_r)
        int n_new0 = 0;
        int slot_r = 0;
        if (lane == 0) slot_r = hash_slot<GL>(sm.keys, cap_mask, shift, rowc, n_new0);
        slot_r = __shfl_sync(FULL_MASK, slot_r, 0);
        double acc_r = 0.0;

        bool nb = false;  // NB: this row logs slots (warp-uniform)
        if (NB) {
            __syncwarp();
            uint4 q0, q1;
            ldg256(rec + 2 * static_cast<int64_t>(rowc), q0, q1);
            const unsigned dr = q0.y;
            if (dr <= static_cast<unsigned>(kNbDeg)) {
                unsigned da = 0, ba = 0;
                int ca = 0;
                if (static_cast<unsigned>(lane) < dr) {
                    ca = tcol[q0.x + lane];
                    uint4 p0, p1;
                    ldg256(rec + 2 * static_cast<int64_t>(ca), p0, p1);
                    da = p0.y;
                    ba = p0.x;
                }
                unsigned incl = da;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned nbv = __shfl_up_sync(FULL_MASK, incl, o);
                    if (lane >= o) incl += nbv;
                }
                const unsigned tot = __shfl_sync(FULL_MASK, incl, 31);
                if (tot <= static_cast<unsigned>(kNbT2)) {
                    const unsigned offa = incl - da;
                    int nn = 0;
                    bool bad = false;
                    if (static_cast<unsigned>(lane) < dr) {
                        nb_off[lane] = static_cast<unsigned short>(offa);
                        const int sl = hash_slot<false>(sm.keys, cap_mask, shift, ca, nn);
                        if (sl < 0) bad = true;
                        else nb_t1[lane] = static_cast<unsigned char>(sl);
                    }
                    __syncwarp();
                    for (unsigned i = 0; i < dr; ++i) {
                        const unsigned di = __shfl_sync(FULL_MASK, da, i);
                        const unsigned bi = __shfl_sync(FULL_MASK, ba, i);
                        const unsigned oi = __shfl_sync(FULL_MASK, offa, i);
                        for (unsigned j = lane; j < di; j += 32) {
                            const int sl = hash_slot<false>(sm.keys, cap_mask, shift, tcol[bi + j], nn);
                            if (sl < 0) bad = true;
                            else nb_t2[oi + j] = static_cast<unsigned char>(sl);
                        }
                        __syncwarp();
                    }
                    const int pre = 1 + warp_sum_int(nn);
                    nb = !__any_sync(FULL_MASK, bad) && pre <= CAPC - CAPC / 4;
                    if (!nb) {  // does not fit: back to an accumulator holding only r
                        for (int i = lane; i < cap; i += 32) sm.keys[i] = EMPTY_KEY;
                        __syncwarp();
                        if (lane == 0) slot_r = hash_slot<false>(sm.keys, cap_mask, shift, rowc, n_new0);
                        slot_r = __shfl_sync(FULL_MASK, slot_r, 0);
                    }
                }
            }
            if (nb && lane < 8) nb_mask[lane] = lane == (slot_r >> 5) ? (1u << (slot_r & 31)) : 0u;
            __syncwarp();
        }
        const int rkey = (NB && nb) ? slot_r : rowc;  // log key of column r
        // split fold for this row (warp-uniform)
        const bool tf = kTF && a.t.tri != nullptr && a.t.tri[rowc] != 0;
        if (kTF && tf) {
            tf_cnt[lane] = 0;
            __syncwarp();
        }

        int distinct = 1;
        bool overflow = false;
        int chains_done = 0;
        int chains_run = N;
        unsigned long long row_steps = 0, row_deg = 0;
        // reference-stream speculation state
        PosT D = 0;
        // first window's stride: L (chains that run to L draw L times; C5's
        // never stop early, C3-heavy's rarely), not 2, which under-delivered
        // and sent the first window of every row dense (C5 10^2 x 32 -15%)
        unsigned ell = LF ? static_cast<unsigned>(LF) : static_cast<unsigned>(a.ell0);
        bool row_done = false;

        while (!row_done) {
            // ------------------------------------------------ walk one batch
            bool active;
            PosT pos = 0;                // next draw index (reference stream)
            int chain = 0;               // chain index (keyed)
            if (IS_REF) {
                active = lane < B;
                pos = D + static_cast<PosT>(lane) * ell;
            } else {
                chain = chains_done + lane;
                active = lane < B && chain < N;
            }
            // step-major log: deposit t of chain (lane) at [t * B + lane], so the
            // walk's writes are bank-conflict free; the fold reads chain-major
            int* lc = sm.log_col + lane;
            double* lw = sm.log_w + lane;
            int m = 0;              // step deposits logged (W0 = 1 at (r, r) is implicit)
            unsigned retm = 0;      // bit t: step deposit t went back to column r (t < 32)
            bool ret_hi = false;    // a return at t >= 32
            double ret_w = 0.0;     // weight of the first return (the only one when L <= 2)
            int state = rowc;
            double w = 1.0;
            unsigned draws = 0;
            unsigned lane_steps = 0, lane_deg = 0;  // committed only if this lane's chain counts
            PosT cached = static_cast<PosT>(~0ull);
            uint4 blk = make_uint4(0, 0, 0, 0);
            bool alive = active;
            bool log_full = false;  // the walk would outgrow this tier's deposit log
            unsigned nb_i1 = 0;     // NB: entry index of the first step in row r
            int k1 = 0;             // split fold: transition index of the first step
#pragma unroll
            for (int t = 0; LF ? (t < LF) : __any_sync(FULL_MASK, alive); ++t) {
                if (LF) {  // compile-time trip count: no log overflow, no length test
                    // (at t = 0 lane 0 is always alive: a batch starts only with chains left)
                    if (t > 0 && !__any_sync(FULL_MASK, alive)) break;
                } else {
                    if (alive && t >= L) alive = false;
                    if (alive && m >= S) {
                        alive = false;
                        log_full = true;
                    }
                }
                if (!alive) continue;
                uint4 r0, r1;
                ldg256(rec + 2 * static_cast<int64_t>(state), r0, r1);
                const unsigned deg = r0.y;
                if (deg == 0) {  // absorbing state (mc_engine.cpp:68)
                    alive = false;
                    continue;
                }
                ++lane_steps;
                if (DEG) lane_deg += deg;
                double ratio;
                int nxt = 0;
                unsigned kidx = 0;  // entry index within the state's row (NB)
                if (deg == 1) {  // forced move, no draw (mc_engine.cpp:69); inline in the record
                    ratio = __hiloint2double(static_cast<int>(r0.w), static_cast<int>(r0.z));
                    nxt = static_cast<int>(r1.z);
                } else {
                    uint32_t ulo, uhi;  // the draw's two words, lo first (rng.hpp:32-41)
                    if (IS_REF) {
                        const PosT b = pos >> 1;
                        if (b != cached) {
                            blk = philox4x32_10_rk(
                                make_uint4(static_cast<uint32_t>(b),
                                           static_cast<uint32_t>(static_cast<unsigned long long>(b) >> 32),
                                           static_cast<uint32_t>(row),
                                           0u),  // row < 2^31: stream id high word
                                a.rk);
                            cached = b;
                        }
                        ulo = (pos & 1) ? blk.z : blk.x;
                        uhi = (pos & 1) ? blk.w : blk.y;
                        ++pos;
                    } else {
                        const PosT b = static_cast<unsigned>(t) >> 1;
                        if (b != cached) {
                            blk = philox4x32_10_rk(
                                make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(chain),
                                           static_cast<uint32_t>(row),
                                           0u),  // row < 2^31: stream id high word
                                a.rk);
                            cached = b;
                        }
                        ulo = (t & 1) ? blk.z : blk.x;
                        uhi = (t & 1) ? blk.w : blk.y;
                    }
                    const double u = u32pair_to_double(ulo, uhi);
                    ++draws;
                    // inverse CDF (mc_engine.cpp:71-77): first k with u < cum_k; the
                    // row's last cum is +inf in the table, which is the reference's
                    // end-1 fallback.  Start at the guide bucket of u, floor(16 u) =
                    // the top 4 bits of the 53-bit draw: every skipped entry has
                    // cum <= m/16 <= u.
                    const unsigned mb = uhi >> 28;
                    const unsigned gw = mb < 8 ? (mb < 4 ? r0.z : r0.w) : (mb < 12 ? r1.x : r1.y);
                    const unsigned g = (gw >> ((mb & 3) * 8)) & 0xffu;
                    unsigned q = r0.x + g * r1.w;  // r1.w = guide scale ceil(deg / 255)
                    double2 e0, e1;
                    if (kAlignedPair) {
                        // Entry pairs are read as one aligned 32-byte load from the
                        // even index at or below the guide start (one L1 request per
                        // pair instead of two).  Starting one entry early is exact:
                        // that entry has cum <= m/16 <= u, or, when it is the
                        // previous row's last entry (odd row begin), it is masked out.
                        q &= ~1u;
                        ldg_pair(ent + q, e0, e1);
                        if (q < r0.x) e0.x = -1.0;  // not this row's: u < -1 is false
                        while (!(u < e0.x) && !(u < e1.x)) {
                            q += 2;
                            ldg_pair(ent + q, e0, e1);
                        }
                    } else {
                        // the first pair resolves almost every draw (16 guide
                        // buckets): selects, not a loop, in the common case
                        e0 = ent[q];
                        e1 = ent[q + 1];  // past the row only when e0 is its +inf entry
                        while (!(u < e0.x) && !(u < e1.x)) {
                            q += 2;
                            e0 = ent[q];
                            e1 = ent[q + 1];
                        }
                    }
                    const bool first_of_pair = u < e0.x;
                    const unsigned k = first_of_pair ? q : q + 1;
                    ratio = first_of_pair ? e0.y : e1.y;
                    kidx = k - r0.x;
                    if (!(NB && nb && t == 1)) nxt = tcol[k];  // NB: the last step logs a slot only
                }
                w *= ratio;  // w *= a_k / p_k (mc_engine.cpp:94)
                int logv;
                if (NB && nb) {
                    if (t == 0) {
                        nb_i1 = kidx;
                        logv = nb_t1[kidx];
                    } else {
                        logv = nb_t2[nb_off[nb_i1] + kidx];
                    }
                    state = nxt;
                } else {
                    state = nxt;
                    logv = state;
                }
                // a lane writes deposit m at step t with m == t (alive lanes never
                // skip a step), so LF kernels index the log with the compile-time t
                const int mi = LF ? t : m;
                if (kTF && tf && t == 0) {
                    k1 = static_cast<int>(kidx);  // counted, not logged (split fold)
                } else {
                    if (LF == 2) {
                        sm.log_col[lf2_col_at(t, lane)] = logv;
                        sm.log_w[lf2_w_at(t, lane)] = w;
                    } else {
                        lc[mi * B] = logv;
                        lw[mi * B] = w;
                    }
                }
                ++m;
                if (logv == rkey) {
                    if (retm == 0 && !ret_hi) ret_w = w;
                    if (LF && LF <= 32) retm |= 1u << t;
                    else if (m <= 32) retm |= 1u << (m - 1);
                    else ret_hi = true;
                }
                // mc_engine.cpp:97 (the last step of a compile-time-L walk needs no test)
                if (!(LF && t == LF - 1) && fabs(w) < a.delta) alive = false;
            }

            if (LF) {  // end-of-chain sentinels for the fold: predicated stores, no loop
#pragma unroll
                for (int t1 = 0; t1 < (LF ? LF : 1); ++t1)
                    if (active && t1 >= m) lc[LF == 2 ? lf2_col_at(t1, lane) - lane : t1 * B] = -1;
            } else if (active) {
                for (int t1 = m; t1 < S; ++t1) lc[t1 * B] = -1;
            }
            if (__any_sync(FULL_MASK, log_full)) {  // longer walks: retry the row on a longer log
                overflow = true;
                break;
            }

            // ------------------------------------------- which lanes count
            unsigned valid;
            const bool first = chains_done == 0;
            const unsigned draws0 = __shfl_sync(FULL_MASK, draws, 0);
            if (first && draws0 == 0) {
                // chain 0 consumed no randomness: its single realization is the
                // estimator mean (mc_engine.cpp:101-104)
                valid = 1u;
                chains_run = 1;
                row_done = true;
            } else if (IS_REF && __all_sync(FULL_MASK, !active || draws == ell)) {
                valid = __ballot_sync(FULL_MASK, active);  // every chain drew ell times: all on the orbit
            } else if (IS_REF) {
                int nxtl = lane;
                if (active && draws > 0) {
                    const unsigned q = draws / ell;
                    if (q * ell == draws && static_cast<unsigned>(lane) + q < static_cast<unsigned>(B))
                        nxtl = lane + static_cast<int>(q);
                }
                unsigned R = (1u << lane) | (1u << nxtl);
                int J = nxtl;
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const unsigned Rn = __shfl_sync(FULL_MASK, R, J);
                    const int Jn = __shfl_sync(FULL_MASK, J, J);
                    R |= Rn;
                    J = Jn;
                }
                valid = __shfl_sync(FULL_MASK, R, 0);
            } else {
                valid = __ballot_sync(FULL_MASK, active);
            }
            const int remaining = N - chains_done;
            if (remaining < 32) valid = lowest_bits(valid, static_cast<int>(remaining));
            const bool mine = (valid >> lane) & 1u;
            if (mine) {
                row_steps += lane_steps;
                row_deg += lane_deg;
            }
            if (IS_REF && !row_done) {
                const int lv = 31 - __clz(valid);
                const unsigned klv = __shfl_sync(FULL_MASK, draws, lv);
                D = D + static_cast<PosT>(lv) * ell + klv;
                // Next stride: prefix speculation (ell = chain 0's draws) yields
                // ~1/p chains per window when a fraction p of chains draw a
                // different count; dense candidates (ell = 1, every draw index)
                // yield B/k.  Go dense when the prefix under-delivers, back to
                // prefix once a dense window shows uniform draw counts.
                const int nv = __popc(valid);
                if (ell > 1 && nv * static_cast<int>(ell) < B) {
                    ell = 1u;
                } else if (ell == 1u) {
                    const bool uniform = __all_sync(FULL_MASK, !((valid >> lane) & 1u) || draws == draws0);
                    if (uniform && draws0 > 1) ell = draws0;
                } else {
                    ell = draws0 > 0 ? draws0 : 1u;
                }
            }
            __syncwarp();

            // split fold: count this batch's first steps per transition of r
            if (kTF && tf) {
                const bool took0 = mine && m >= 1;
                const unsigned pk = __match_any_sync(FULL_MASK, took0 ? k1 : -1 - lane);
                // ordered before the next batch's updates and the row-end read
                // by the fold's __syncwarp()s
                if (took0 && (pk & lt_mask) == 0) tf_cnt[k1] += __popc(pk);
            }
            // ------------------------------------- ordered (chain, step) fold
            // (i) column r: W0 = +1.0 per valid chain plus its returns, in
            // chain order, folded in a register (warp-uniform).
            {
                const unsigned rl = __ballot_sync(FULL_MASK, mine && (retm != 0 || ret_hi));
                if (rl == 0) {
                    acc_r = add_ones(acc_r, __popc(valid));
                } else {
                    // L <= 2: a chain returns to r at most once (A has no self loops,
                    // so only its last step can land on r)
                    constexpr bool kMulti = LF == 0 || LF > 2;
                    const unsigned multi =
                        kMulti ? __ballot_sync(FULL_MASK, mine && ((retm & (retm - 1)) != 0 || ret_hi)) : 0u;
                    // W0 additions owed before this lane's return: valid chains after
                    // the previous returning lane, up to and including this one
                    const unsigned prevs = rl & lt_mask;
                    const unsigned prev_mask = prevs ? ((2u << (31 - __clz(prevs))) - 1u) : 0u;
                    const int run = __popc(valid & lt_mask & ~prev_mask) + 1;
                    unsigned todo = rl;
                    while (todo) {
                        const int j = __ffs(todo) - 1;
                        todo &= todo - 1;
                        acc_r = add_ones(acc_r, __shfl_sync(FULL_MASK, run, j));
                        acc_r += __shfl_sync(FULL_MASK, ret_w, j);  // first return of chain j
                        if (kMulti && ((multi >> j) & 1u)) {  // later returns of chain j, in step order
                            const unsigned rm = __shfl_sync(FULL_MASK, retm, j);
                            const bool hi = __shfl_sync(FULL_MASK, static_cast<int>(ret_hi), j) != 0;
                            unsigned rest = rm & (rm - 1);
                            while (rest) {
                                const int t1 = __ffs(rest) - 1;
                                rest &= rest - 1;
                                acc_r += sm.log_w[t1 * B + j];
                            }
                            if (hi) {  // returns at steps >= 32 (max_len > 32 only)
                                bool skip = rm == 0;  // the first return was at a step >= 32
                                const int mj = __shfl_sync(FULL_MASK, m, j);
                                for (int t1 = 32; t1 < mj; ++t1)
                                    if (sm.log_col[t1 * B + j] == rowc) {
                                        if (skip) skip = false;
                                        else acc_r += sm.log_w[t1 * B + j];
                                    }
                            }
                        }
                    }
                    const int last = 31 - __clz(rl);
                    const unsigned upto = last == 31 ? FULL_MASK : ((2u << last) - 1u);
                    acc_r = add_ones(acc_r, __popc(valid & ~upto));
                }
            }
            // (ii) every other column: 32-position chunks of the chain-major log;
            // equal columns grouped by __match_any_sync; the group's left fold runs
            // as a shuffle chain in lane (= chain-major) order.
            int n_new = 0;
            bool fail = false;
            // split fold: only the step-1 deposits (position p = chain j, step 1)
            const int span = (kTF && tf) ? B : B * S;
            for (int base = 0; base < span; base += 32) {
                const int p = base + lane;
                // chain of position p: p / S (shift for power-of-two S, else the magic multiply)
                const int j = (kTF && tf) ? p
                                          : min(s_shift >= 0 ? (p >> s_shift)
                                                             : static_cast<int>(
                                                                   __umulhi(static_cast<unsigned>(p), a.log_magic)),
                                                31);
                bool ok = p < span && ((valid >> j) & 1u);
                // chain-major position p -> step-major slot
                const int q = (kTF && tf) ? B + j : (p - j * S) * B + j;
                const int tq = (kTF && tf) ? 1 : p - j * S;  // step of position p
                int c = ok ? sm.log_col[LF == 2 ? lf2_col_at(tq, j) : q] : -1;
                ok = ok && c >= 0 && c != rkey;  // column r was folded in (i)
                if (!ok) c = -1 - lane;          // unique non-column tag
                const unsigned peers = __match_any_sync(FULL_MASK, c);
                // group rank = position of this entry among equal columns of the
                // chunk (lane order == chain-major order); predecessor = the
                // previous entry of the group
                const unsigned below = peers & lt_mask;
                const int rank = __popc(below);
                const int pred = below ? 31 - __clz(below) : lane;
                const int gsize = ok ? __popc(peers) : 0;
                const int leader = __ffs(peers) - 1;
                int slot = 0;
                bool fresh = false;  // the leader inserted the column: its value is 0.0
                if (ok && rank == 0) {
                    if (NB && nb) {
                        slot = c;
                        atomicOr(&nb_mask[c >> 5], 1u << (c & 31));
                    } else {
                        const int had = n_new;
                        slot = hash_slot<GL>(sm.keys, cap_mask, shift, c, n_new);
                        fresh = n_new != had;
                        if (slot < 0) fail = true;
                    }
                }
                if (NB && nb) slot = ok ? c : 0;  // the logged key is the slot
                else slot = __shfl_sync(FULL_MASK, slot, leader);
                const double w = ok ? sm.log_w[LF == 2 ? lf2_w_at(tq, j) : q] : 0.0;
                double v = w;
                // an empty slot holds 0.0 (the accumulator invariant): a fresh
                // column skips the load (HBM latency on the global tiers)
                if (ok && rank == 0 && slot >= 0) v = (GL && fresh ? 0.0 : sm.vals[slot]) + w;
                const int maxsize = __reduce_max_sync(FULL_MASK, static_cast<unsigned>(gsize));
#pragma unroll 2
                for (int it = 1; it < maxsize; ++it) {  // left fold along each group, one link per round
                    const double prev = __shfl_sync(FULL_MASK, v, pred);
                    if (rank == it) v = prev + w;
                }
                if (ok && slot >= 0 && rank == gsize - 1) sm.vals[slot] = v;
                __syncwarp();
            }
            distinct += warp_sum_int(n_new);
            if (__any_sync(FULL_MASK, fail) || distinct > (CAPC ? CAPC - CAPC / 4 : a.cap_limit)) {
                overflow = true;
                break;
            }
            chains_done += __popc(valid);
            if (chains_done >= N) row_done = true;
        }

        if (kTF && tf && !overflow) {
            // split fold: column c_k = m_k sequential additions of ratio_k, in
            // chain order (all equal, so only the count matters); c_k was never
            // touched by a step-1 deposit, so this inserts it
            uint4 q0, q1;
            ldg256(rec + 2 * static_cast<int64_t>(rowc), q0, q1);
            int nn = 0;
            bool bad = false;
            if (static_cast<unsigned>(lane) < q0.y) {
                const int mk = tf_cnt[lane];
                if (mk > 0) {
                    const double rk = ent[q0.x + lane].y;
                    double v = 0.0;
#pragma unroll 4
                    for (int i = 0; i < mk; ++i) v += rk;  // mc_engine.cpp:49, chain order
                    const int sl = hash_slot<GL>(sm.keys, cap_mask, shift, tcol[q0.x + lane], nn);
                    if (sl < 0) bad = true;
                    else sm.vals[sl] = v;
                }
            }
            distinct += warp_sum_int(nn);
            if (__any_sync(FULL_MASK, bad) || distinct > (CAPC ? CAPC - CAPC / 4 : a.cap_limit)) overflow = true;
            __syncwarp();
        }
        const int64_t lrow = static_cast<int64_t>(row) - a.row_begin;
        if (overflow) {
            if (lane == 0) {
                const unsigned long long q = atomicAdd(&a.counters[3], 1ull);
                a.overflow_list[q] = rowc;
            }
            for (int i = lane; i < cap; i += 32) {
                sm.keys[i] = EMPTY_KEY;
                sm.vals[i] = 0.0;
            }
            __syncwarp();
            continue;
        }
        tot_steps += row_steps;
        tot_deg += row_deg;
        if (lane == 0) sm.vals[slot_r] = acc_r;
        unsigned nb_bits = 0;  // NB: lane l < 8 holds touched-mask word l
        if (NB && nb) {
            nb_bits = lane < 8 ? nb_mask[lane] : 0u;
            distinct = warp_sum_int(__popc(nb_bits));
        }
        __syncwarp();

        // ------------------------------------------------------ finalize
        // compact occupied slots to [0, s) in place, emptying the vacated slots
        int o = 0;
        // GL: 4 chunks of slots loaded per round (HBM latency); the writes of a
        // round go to slots that round (or an earlier one) already read
        constexpr int CU = GL ? 4 : 1;
        for (int g0 = 0; g0 < cap; g0 += 32 * CU) {
            int kk[CU];
            double vv[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) {
                const int i = g0 + 32 * u + lane;
                kk[u] = i < cap ? sm.keys[i] : EMPTY_KEY;
                vv[u] = i < cap ? sm.vals[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < CU; ++u) {
                const int i0 = g0 + 32 * u;
                const int i = i0 + lane;
                bool occ = kk[u] != EMPTY_KEY;
                bool drop = false;  // NB: pre-inserted but never visited
                if (NB && nb) {
                    const unsigned wbits = __shfl_sync(FULL_MASK, nb_bits, i0 >> 5);
                    drop = occ && !((wbits >> lane) & 1u);
                    occ = occ && !drop;
                }
                const unsigned bal = __ballot_sync(FULL_MASK, occ);
                const int dst = o + __popc(bal & lt_mask);
                __syncwarp();
                if ((occ && dst != i) || drop) {
                    sm.keys[i] = EMPTY_KEY;
                    sm.vals[i] = 0.0;
                }
                __syncwarp();
                if (occ) {
                    sm.keys[dst] = kk[u];
                    sm.vals[dst] = vv[u];
                }
                o += __popc(bal);
                __syncwarp();
            }
        }
        const int s = distinct;
        const double inv_n = 1.0 / static_cast<double>(chains_run);  // mc_engine.cpp:109
        if (GL) {
            for (int g0 = lane; g0 < s; g0 += 128) {
                double vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) vv[u] = g0 + 32 * u < s ? sm.vals[g0 + 32 * u] : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (g0 + 32 * u < s) sm.vals[g0 + 32 * u] = vv[u] * inv_n;
            }
        } else {
            for (int i = lane; i < s; i += 32) sm.vals[i] = sm.vals[i] * inv_n;
        }
        __syncwarp();

        const int64_t kret = a.retain_k;
        bool keep_all = kret <= 0 || static_cast<int64_t>(s) <= kret;
        int len = s;        // entries that go to the output stage (column-sorted)
        int touched = s;    // slots [0, touched) to restore to empty afterwards
        if (!keep_all && s > kRankTopkMax) {
            // retain_top_k by radix selection, then sort only the kept entries
            unsigned* hist = reinterpret_cast<unsigned*>(sm.vals + (cap - 128));  // free: s <= 3/4 cap
            unsigned long long T;
            int Tc, copied;
            radix_topk(sm.keys, sm.vals, s, static_cast<int>(kret), rowc, hist, cap - 128 - s, T, Tc, copied);
            for (int b = lane; b < 256; b += 32) hist[b] = 0;  // restore the zeros of the vals array
            for (int i = s + lane; i < s + copied; i += 32) {  // and empty the candidates' copies
                sm.keys[i] = EMPTY_KEY;
                sm.vals[i] = 0.0;
            }
            __syncwarp();
            int kept = 0;
            for (int g0 = 0; g0 < s; g0 += 128) {  // stable forward compaction of the kept set
                int kk[4];
                double vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = g0 + 32 * u + lane;
                    kk[u] = i < s ? sm.keys[i] : rowc;
                    vv[u] = i < s ? sm.vals[i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    bool keep = false;
                    if (g0 + 32 * u + lane < s) {
                        const unsigned long long key = topk_key(kk[u], vv[u], rowc);
                        keep = key > T || (key == T && kk[u] <= Tc);
                    }
                    const unsigned bal = __ballot_sync(FULL_MASK, keep);
                    __syncwarp();
                    if (keep) {
                        sm.keys[kept + __popc(bal & lt_mask)] = kk[u];
                        sm.vals[kept + __popc(bal & lt_mask)] = vv[u];
                    }
                    kept += __popc(bal);
                    __syncwarp();
                }
            }
            len = kept;
            keep_all = true;
            touched = max(touched, sort_by_column(sm.keys, sm.vals, len));
        } else {
            touched = max(touched, sort_by_column(sm.keys, sm.vals, s));
        }

        const int64_t out_off = a.stage_base + static_cast<int64_t>(wi) * a.stage_stride;
        int* __restrict__ oc = a.stage_col + out_off;
        double* __restrict__ ov = a.stage_val + out_off;
        int n_out = 0;
        for (int i0 = 0; i0 < len; i0 += 32) {
            const int i = i0 + lane;
            bool keep = i < len;
            int c = 0;
            double v = 0.0;
            if (keep) {
                c = sm.keys[i];
                v = sm.vals[i];
                if (!keep_all) {  // small rows: rank in retain_top_k order
                    int64_t rank = 0;
                    for (int j = 0; j < len; ++j) rank += topk_before(sm.keys[j], sm.vals[j], c, v, rowc);
                    keep = rank < kret;
                }
            }
            if (keep && !a.unscaled) {
                v = v / a.t.b1_diag[c];                // scale_columns (mc_engine.cpp:148)
                keep = !(v == 0.0 && c != rowc);       // prune (mc_engine.cpp:174-176)
            }
            const unsigned bal = __ballot_sync(FULL_MASK, keep);
            if (keep) {
                const int dst = n_out + __popc(bal & lt_mask);
                oc[dst] = c;
                ov[dst] = v;
            }
            n_out += __popc(bal);
        }
        if (lane == 0) {
            a.row_cnt[lrow] = n_out;
            a.row_src[lrow] = out_off;
            a.chains_used[lrow] = chains_run;
            a.entries_before[lrow] = s;
        }
        __syncwarp();
        for (int i = lane; i < touched; i += 32) {  // back to an empty accumulator
            sm.keys[i] = EMPTY_KEY;
            sm.vals[i] = 0.0;
        }
        __syncwarp();
    }

    tot_steps = warp_sum_u64(tot_steps);
    tot_deg = warp_sum_u64(tot_deg);
    if (lane == 0) {
        atomicAdd(&a.counters[1], tot_steps);
        atomicAdd(&a.counters[2], tot_deg);
    }
}

}  // namespace

size_t walk_smem_bytes_per_warp(int cap, int lanes, int log_stride) {
    return static_cast<size_t>(cap + round32(lanes * log_stride)) * 12;
}

size_t walk_global_bytes_per_warp(int cap, int lanes, int log_stride) {
    return walk_smem_bytes_per_warp(cap, lanes, log_stride);
}

template <int MODE, int MINB, bool GL, bool DEG, int LF = 0, int CAPC = 0, bool NB = false>
cudaError_t launch_walk_t(const WalkArgs& a, int warps_per_block, int num_sms, int64_t max_warps,
                          cudaStream_t s) {
    const size_t smem =
        GL ? 0
           : (walk_smem_bytes_per_warp(a.cap, a.lanes, a.log_stride) + (NB ? kNbBytes : 0) +
              (split_fold_kernel<LF, NB>() ? kTfBytes : 0)) *
                 warps_per_block;
    const int threads = warps_per_block * 32;
    cudaError_t e = cudaFuncSetAttribute(k_walk<MODE, MINB, GL, DEG, LF, CAPC, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_walk<MODE, MINB, GL, DEG, LF, CAPC, NB>, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t blocks = static_cast<int64_t>(per_sm) * num_sms;
    const int64_t need = (a.n_work + warps_per_block - 1) / warps_per_block;
    if (blocks > need) blocks = need;
    if (max_warps > 0 && blocks * warps_per_block > max_warps)
        blocks = std::max<int64_t>(1, max_warps / warps_per_block);
    k_walk<MODE, MINB, GL, DEG, LF, CAPC, NB><<<static_cast<unsigned>(blocks), threads, smem, s>>>(a);
    return cudaGetLastError();
}

// MCMI_WALK_MINB (env, tuning only) selects the __launch_bounds__ min-blocks
// variant: 4 = 64 regs (32 warps/SM), 5 = 48 regs (40 warps), 6 = 40 regs (48 warps).
int walk_minb() {
    static int v = [] {
        const char* e = getenv("MCMI_WALK_MINB");
        const int x = e ? atoi(e) : kDefaultMinBlocks;
        return (x == 4 || x == 5 || x == 6) ? x : kDefaultMinBlocks;
    }();
    return v;
}

// Neighbourhood slot tables for the L = 2 kernels: the host's cost hint
// (WalkArgs::nb_hint), overridden by MCMI_WALK_NB=0 / 1 (tuning and tests).
bool walk_nb(const WalkArgs& a) {
    const char* e = getenv("MCMI_WALK_NB");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    return a.nb_hint != 0;
}

// The compile-time (walk length, capacity) variants of k_walk for MODE 0 / 1;
// false if none fits this launch (lanes must be 32 and log_stride == L).
template <int MODE>
bool launch_specialised(const WalkArgs& a, int wpb, int sms, cudaStream_t s, cudaError_t* err) {
    if (a.lanes != 32 || a.log_stride != a.max_len) return false;
    switch (a.max_len) {
        case 2:
            if (walk_nb(a) && (a.cap == 32 || a.cap == 64 || a.cap == 256)) {
                *err = a.cap == 32   ? launch_walk_t<MODE, 6, false, false, 2, 32, true>(a, wpb, sms, 0, s)
                       : a.cap == 64 ? launch_walk_t<MODE, 6, false, false, 2, 64, true>(a, wpb, sms, 0, s)
                                     : launch_walk_t<MODE, 6, false, false, 2, 256, true>(a, wpb, sms, 0, s);
                return true;
            }
            *err = a.cap == 32    ? launch_walk_t<MODE, 6, false, false, 2, 32>(a, wpb, sms, 0, s)
                   : a.cap == 64  ? launch_walk_t<MODE, 6, false, false, 2, 64>(a, wpb, sms, 0, s)
                   : a.cap == 256 ? launch_walk_t<MODE, 6, false, false, 2, 256>(a, wpb, sms, 0, s)
                                  : launch_walk_t<MODE, 6, false, false, 2>(a, wpb, sms, 0, s);
            return true;
        case 3:
            *err = a.cap == 256 ? launch_walk_t<MODE, 6, false, false, 3, 256>(a, wpb, sms, 0, s)
                                : launch_walk_t<MODE, 6, false, false, 3>(a, wpb, sms, 0, s);
            return true;
        case 4:
            *err = a.cap == 256 ? launch_walk_t<MODE, 6, false, false, 4, 256>(a, wpb, sms, 0, s)
                                : launch_walk_t<MODE, 6, false, false, 4>(a, wpb, sms, 0, s);
            return true;
        case 8:
            *err = a.cap == 256 ? launch_walk_t<MODE, 6, false, false, 8, 256>(a, wpb, sms, 0, s)
                                : launch_walk_t<MODE, 6, false, false, 8>(a, wpb, sms, 0, s);
            return true;
        default:
            return false;
    }
}

cudaError_t launch_walk(const WalkArgs& a_in, int warps_per_block, int num_sms, bool global_tier,
                        int64_t max_warps, cudaStream_t s) {
    if (a_in.n_work <= 0) return cudaSuccess;
    WalkArgs a = a_in;  // derived per-launch constants, so the kernel re-reads rather than recomputes them
    {  // Philox round keys of the master seed (rng.hpp:56-66 key schedule)
        uint32_t k0 = static_cast<uint32_t>(a.seed), k1 = static_cast<uint32_t>(a.seed >> 32);
        for (int r = 0; r < 10; ++r, k0 += 0x9E3779B9u, k1 += 0xBB67AE85u) {
            a.rk[2 * r] = k0;
            a.rk[2 * r + 1] = k1;
        }
    }
    a.log_n = round32(a.lanes * a.log_stride);
    a.warp_bytes = static_cast<long long>(walk_smem_bytes_per_warp(a.cap, a.lanes, a.log_stride));
    {
        int lg = 0;
        while ((1 << lg) < a.cap) ++lg;
        a.hash_shift = 32 - lg;
        const int S = a.log_stride;
        int ls = -1;
        if ((S & (S - 1)) == 0) {
            ls = 0;
            while ((1 << ls) < S) ++ls;
        }
        a.log_shift = ls;
    }
    const int mb = walk_minb();
    const bool pos64 = static_cast<double>(a.n_chains) * static_cast<double>(std::max<int64_t>(a.max_len, 1)) >=
                           4294967295.0 ||  // draw positions beyond 32 bits
                       getenv("MCMI_FORCE_POS64") != nullptr;  // tests exercise the 64-bit variant
    const int mode = a.rng_mode == 0 ? (pos64 ? 2 : 0) : 1;
    // Walk-length specialisations (compile-time step loop and fold arithmetic,
    // plus compile-time hash capacity for the common tiers): L = 2 (every
    // defaults config), 3, 4 and 8 (C5).  Measured -2..-14% against the generic
    // kernel.  MCMI_WALK_GENERIC (tuning) disables them.
    const bool spec = getenv("MCMI_WALK_GENERIC") == nullptr;
    cudaError_t se = cudaSuccess;
    // variants: the global tier and the statistics build use one launch bound
    if (mode == 2) {
        if (global_tier)
            return a.deg_stats ? launch_walk_t<2, kGlMinBlocks, true, true>(a, warps_per_block, num_sms, max_warps, s)
                               : launch_walk_t<2, kGlMinBlocks, true, false>(a, warps_per_block, num_sms, max_warps, s);
        if (a.deg_stats) return launch_walk_t<2, 6, false, true>(a, warps_per_block, num_sms, 0, s);
        return launch_walk_t<2, 6, false, false>(a, warps_per_block, num_sms, 0, s);
    }
    if (mode == 0) {
        if (global_tier)
            return a.deg_stats ? launch_walk_t<0, kGlMinBlocks, true, true>(a, warps_per_block, num_sms, max_warps, s)
                               : launch_walk_t<0, kGlMinBlocks, true, false>(a, warps_per_block, num_sms, max_warps, s);
        if (a.deg_stats) return launch_walk_t<0, 6, false, true>(a, warps_per_block, num_sms, 0, s);
        if (mb == 5) return launch_walk_t<0, 5, false, false>(a, warps_per_block, num_sms, 0, s);
        if (mb == 4) return launch_walk_t<0, 4, false, false>(a, warps_per_block, num_sms, 0, s);
        if (spec && launch_specialised<0>(a, warps_per_block, num_sms, s, &se)) return se;
        return launch_walk_t<0, 6, false, false>(a, warps_per_block, num_sms, 0, s);
    }
    if (global_tier)
        return a.deg_stats ? launch_walk_t<1, kGlMinBlocks, true, true>(a, warps_per_block, num_sms, max_warps, s)
                           : launch_walk_t<1, kGlMinBlocks, true, false>(a, warps_per_block, num_sms, max_warps, s);
    if (a.deg_stats) return launch_walk_t<1, 6, false, true>(a, warps_per_block, num_sms, 0, s);
    if (mb == 5) return launch_walk_t<1, 5, false, false>(a, warps_per_block, num_sms, 0, s);
    if (mb == 4) return launch_walk_t<1, 4, false, false>(a, warps_per_block, num_sms, 0, s);
    if (spec && launch_specialised<1>(a, warps_per_block, num_sms, s, &se)) return se;
    return launch_walk_t<1, 6, false, false>(a, warps_per_block, num_sms, 0, s);
}

}  // namespace mcmi
