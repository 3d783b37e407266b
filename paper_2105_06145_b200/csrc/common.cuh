// common.cuh — device building blocks shared by the round loop and the standalone
// LaB-PQ: memory-order helpers, warp-aggregated compaction, the grid barrier, the
// counter-based sampler and the CTA-wide radix selection used for ExtDist.
//
// Citations: P:n = /root/reference/PAPER.md line n.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sssp.h"

namespace sssp {

constexpr uint64_t kInf = 0xFFFFFFFFFFFFFFFFull;
constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kMaxSamples = 65536;  // cap on the theta sample count s (reading R5)

// ------------------------------------------------------------------ loads / stores
// delta[] is written by atomics that resolve in L2; reads that decide membership
// (Extract) or filter relaxations go to L2 (.cg) so a stale L1 line can never be
// observed within the persistent kernel.
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) { return __ldcg((const unsigned long long*)p); }
__device__ __forceinline__ int32_t ld_cg_i32(const int32_t* p) { return __ldcg(p); }
// streaming, read-only CSR (never written during a run): keep it out of L1.
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// CSR row bounds off[i], off[i+1] in one 8-byte-or-two load pair, issued in program order
// (asm volatile) so that it stays ahead of a following atom_or_u64 instead of being sunk
// below the branch on the atomic's result
__device__ __forceinline__ void ld_row(const int32_t* off, int32_t i, int32_t& beg, int32_t& end) {
    asm volatile("ld.global.nc.s32 %0, [%2];\n\tld.global.nc.s32 %1, [%2+4];" : "=r"(beg), "=r"(end) : "l"(off + i));
}
// 16-byte global -> shared copy through L2 (no register holds the data in between)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint64_t atom_or_u64(uint64_t* p, uint64_t x) {
    uint64_t old;
    asm volatile("atom.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(x) : "memory");
    return old;
}
// one interleaved arc {head, weight}: a single 8-byte load (one row, one TLB lookup)
__device__ __forceinline__ uint2 ld_stream_arc(const uint2* p) {
    uint2 a;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(a.x), "=r"(a.y) : "l"(p));
    return a;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const unsigned* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) { return *(volatile const uint64_t*)p; }
__device__ __forceinline__ int32_t ld_volatile_i32(const int32_t* p) { return *(volatile const int32_t*)p; }
__device__ __forceinline__ int64_t ld_volatile_i64(const int64_t* p) { return *(volatile const int64_t*)p; }
__device__ __forceinline__ int32_t ld_acquire_i32(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_i32(int32_t* p, int32_t v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// WriteMin: atomic min, true iff it strictly decreased *p.
__device__ __forceinline__ uint64_t atomic_min_u64(uint64_t* p, uint64_t v) {
    return atomicMin((unsigned long long*)p, (unsigned long long)v);
}

// Warp-aggregated append of the lanes with `pred` to out[*cursor ...].
// All 32 lanes must call it.  Returns this lane's slot (or -1).
__device__ __forceinline__ int32_t warp_append_slot(bool pred, int32_t* cursor) {
    uint32_t mask = __ballot_sync(kFull, pred);
    if (mask == 0) return -1;
    int leader = __ffs(mask) - 1;
    int32_t base = 0;
    if (lane_id() == leader) base = atomicAdd(cursor, __popc(mask));
    base = __shfl_sync(kFull, base, leader);
    return pred ? base + __popc(mask & lanemask_lt()) : -1;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t t = __shfl_xor_sync(kFull, v, o);
        v = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t t = __shfl_xor_sync(kFull, v, o);
        v = t > v ? t : v;
    }
    return v;
}
__device__ __forceinline__ int32_t warp_incl_scan(int32_t v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(kFull, v, o);
        if (lane_id() >= o) v += t;
    }
    return v;
}

// Exclusive warp prefix sum of values in [0, 2^BITS) by bit-plane ballots: BITS
// independent ballot + popc pairs instead of five dependent shuffles (this sits on the
// dependency chain of every relax step).  `total` = the warp sum.
template <int BITS>
__device__ __forceinline__ int32_t warp_excl_scan_small(int32_t v, int32_t& total) {
    const uint32_t lt = lanemask_lt();
    int32_t ex = 0, tot = 0;
#pragma unroll
    for (int b = 0; b < BITS; b++) {
        const uint32_t m = __ballot_sync(kFull, (v >> b) & 1);
        ex += __popc(m & lt) << b;
        tot += __popc(m) << b;
    }
    total = tot;
    return ex;
}

// ------------------------------------------------------------------ grid barrier
// Requires a cooperative launch.  cooperative_groups' grid sync measured 1.2 us at
// 296-444 CTAs on B200 vs 1.5-1.9 us for a hand-written arrive/spin counter
// (scripts/bench_barrier.cu, profiles/bench_barrier_r1.log).
// (no counter argument: the hand-written arrive/spin barrier was replaced by this one)
__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }

// ------------------------------------------------------------------ sampling (reading R5/R6)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// s = ceil(10 q / rho) + 10 (1 + floor(log2(q + 1))), capped (reading R5)
__host__ __device__ __forceinline__ uint64_t sample_count(uint64_t q, uint64_t rho) {
    uint64_t lg = 0;
    for (uint64_t x = q + 1; x > 1; x >>= 1) lg++;
    uint64_t s = (10 * q + rho - 1) / rho + 10 * (1 + lg);
    return s > (uint64_t)kMaxSamples ? (uint64_t)kMaxSamples : s;
}

// key accessors for cta_kth_smallest
struct QueueKey {  // key of the i-th queued id: keys[queue[i]] (read through L2)
    const int32_t* queue;
    const uint64_t* keys;
    __device__ uint64_t operator()(int64_t i) const { return ld_cg_u64(keys + ld_cg_i32(queue + i)); }
};
struct ArrayKey {
    const uint64_t* a;
    __device__ uint64_t operator()(int64_t i) const { return a[i]; }
};

// ------------------------------------------------------------------ CTA radix select
// k-th smallest (1-based) of `count` keys produced by key(i), computed by one CTA.
// MSD radix select over the bits where min and max differ, 8 bits per pass.
struct SelectSmem {
    uint32_t hist[256];
    uint64_t red[32];
    uint64_t bcast[2];
};

template <typename KeyFn>
__device__ uint64_t cta_kth_smallest(KeyFn key, int64_t count, uint64_t k, SelectSmem& sm) {
    const int tid = threadIdx.x, nthr = blockDim.x, nw = (nthr + 31) / 32, wid = tid >> 5;
    // min / max
    uint64_t lo = kInf, hi = 0;
    for (int64_t i = tid; i < count; i += nthr) {
        uint64_t x = key(i);
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    }
    lo = warp_min_u64(lo);
    hi = warp_max_u64(hi);
    if (lane_id() == 0) sm.red[wid] = lo;
    __syncthreads();
    if (tid == 0) {
        uint64_t a = kInf;
        for (int w = 0; w < nw; w++) a = sm.red[w] < a ? sm.red[w] : a;
        sm.bcast[0] = a;
    }
    __syncthreads();
    lo = sm.bcast[0];
    __syncthreads();
    if (lane_id() == 0) sm.red[wid] = hi;
    __syncthreads();
    if (tid == 0) {
        uint64_t a = 0;
        for (int w = 0; w < nw; w++) a = sm.red[w] > a ? sm.red[w] : a;
        sm.bcast[1] = a;
    }
    __syncthreads();
    hi = sm.bcast[1];
    if (lo == hi) return lo;
    const int top = 63 - __clzll((long long)(lo ^ hi));  // highest differing bit
    uint64_t prefix = (top == 63) ? 0 : (lo >> (top + 1)) << (top + 1);
    int sh = top + 1;
    while (sh > 0) {
        const int nb = sh >= 8 ? 8 : sh;
        sh -= nb;
        const int above = sh + nb;  // bits >= above must equal prefix
        const uint64_t mask_above = above >= 64 ? 0 : ~((1ull << above) - 1);
        for (int b = tid; b < 256; b += nthr) sm.hist[b] = 0;
        __syncthreads();
        for (int64_t i = tid; i < count; i += nthr) {
            uint64_t x = key(i);
            if ((x & mask_above) == prefix) atomicAdd(&sm.hist[(x >> sh) & ((1u << nb) - 1)], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // warp 0: each lane owns 8 consecutive bins
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                c[j] = sm.hist[tid * 8 + j];
                tot += c[j];
            }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(kFull, incl, o);
                if (tid >= o) incl += t;
            }
            uint32_t excl = incl - tot;
            bool mine = (uint64_t)excl < k && k <= (uint64_t)incl;
            if (mine) {
                uint64_t kk = k - excl;
                int d = 0;
                for (int j = 0; j < 8; j++) {
                    if (kk <= c[j]) {
                        d = tid * 8 + j;
                        break;
                    }
                    kk -= c[j];
                }
                sm.bcast[0] = prefix | ((uint64_t)d << sh);
                sm.bcast[1] = kk;
            }
        }
        __syncthreads();
        prefix = sm.bcast[0];
        k = sm.bcast[1];
        __syncthreads();
    }
    return prefix;
}

}  // namespace sssp
