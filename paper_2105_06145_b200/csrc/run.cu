// run.cu — the stepping-algorithm round loop (Alg. 1) as ONE persistent
// cooperative kernel, plus the sssp_* handle API.
//
// LaB-PQ of the round loop (DESIGN.md §5 "Queue state"): the membership flag of a
// vertex lives in the top bit of its delta word (bit 63 set = NOT in Q), the value
// in the low 63 bits; the queue is a compacted id array (ping-pong per round).
//   Update(v)   = the WriteMin CAS that lowers the value also clears bit 63; the
//                 thread whose CAS saw bit 63 set appends v (exactly one append per
//                 insertion, no duplicates).
//   Extract(u)  = atomicOr(bit 63): deletes u from Q and returns, atomically, the
//                 value it is relaxed with (its snapshot key).
// Because flag and key share one word, a concurrent WriteMin and Extract can never
// lose an update, so Extract and relax may overlap ("live" rounds, the default).
//
// Per round r:
//   ExtDist  theta_r per policy (Table tab:framework).  rho: every CTA
//            draws the same counter-based samples into shared memory and radix-
//            selects the same theta (readings R5/R6) -> no barrier.
//   Phase A  one pass over the queue (array LaB-PQ P:1011-1012): ids with
//            key <= theta are extracted; vertices of degree <= kLight are relaxed at
//            once by the extracting warp (live) or listed (snapshot mode); heavier
//            ones are cut into kChunk-arc descriptors; the rest of Q is compacted
//            into the next queue.                                     grid barrier
//   Phase B  warps stride over the chunk descriptors (and, in snapshot mode, the
//            light list): per arc c = d_u + w, plain L2 load filter, WriteMin by
//            CAS, append on insertion.       grid barrier (only if non-empty)
//   loop while |Q| > 0: |Q_{r+1}| is the next queue's tail counter.
#include <stdio.h>

#include <algorithm>
#include <string.h>

#include "common.cuh"
#include "internal.h"

namespace sssp {

constexpr uint64_t kTop = 1ull << 63;  // flag bit: set = not in Q
constexpr uint64_t kVal = kTop - 1;    // value bits of a delta word
#ifndef SSSP_MIN_BLOCKS
#define SSSP_MIN_BLOCKS 2
#endif
#ifndef SSSP_ARCS
#define SSSP_ARCS 8
#endif
#ifndef SSSP_LIGHT
#define SSSP_LIGHT 128
#endif
constexpr int kBlock = 512;                 // threads per CTA of the round loop
constexpr int kMinBlocks = SSSP_MIN_BLOCKS; // CTAs per SM the register budget targets
constexpr int kArcs = SSSP_ARCS;            // arcs per lane in flight
constexpr int kChunk = 32 * kArcs;     // arcs per heavy-chunk descriptor
constexpr int kLight = SSSP_LIGHT;     // out-degree <= kLight: relaxed by the extracting warp
constexpr int kSmemSamples = 4096;     // theta samples held in shared memory (else CTA-0 fallback)
constexpr int kRankSelect = 256;       // s <= this: select by rank counting

// A vertex (or a piece of one) to relax: snapshot key and a CSR arc range.
struct __align__(16) Desc {
    uint64_t d;
    int32_t beg;
    int32_t len;
};

struct __align__(128) RoundCnt {
    int32_t tail;    // next-queue write cursor (remaining ids, then inserted ids)
    int32_t nlight;  // snapshot mode: light frontier entries
    int32_t nchunk;  // heavy chunk descriptors
    int32_t nheavy;  // STATS: heavy vertices
    unsigned long long minrem;   // min key among ids Extract kept in Q
    unsigned long long minsucc;  // min successful WriteMin value
    unsigned long long theta;    // CTA-0 fallback theta
    unsigned long long fsize;    // STATS: extracted
    unsigned long long edges;    // STATS: arcs of extracted vertices
    unsigned long long succ;     // STATS: successful WriteMins
    unsigned long long inserts;  // STATS: ids appended by relax
    unsigned long long pad[5];
};

struct __align__(128) Ctrl {
    unsigned bar;  // grid barrier arrival counter
    unsigned pad0[31];
    RoundCnt cnt[3];
    // results (copied to the host after the run)
    int32_t status;
    int32_t pad1;
    int64_t rounds;
    int64_t tot_extracted, tot_edges, tot_succ, tot_inserts, tot_qscan, max_q, max_f;
};

struct RunParams {
    int32_t n;
    int32_t source;
    int64_t m;
    const int32_t* __restrict__ off;
    const int32_t* __restrict__ idx;
    const uint32_t* __restrict__ w;
    uint64_t* dist;
    int32_t* q0;
    int32_t* q1;
    Desc* light;
    Desc* chunks;
    uint64_t* samples;
    Ctrl* ctrl;
    uint64_t param;
    uint32_t flags;
    uint64_t seed;
    int64_t max_rounds;
    sssp_round* trace;
    int64_t trace_cap;
    int32_t* ext_count;
};

__device__ __forceinline__ void reset_cnt(RoundCnt* c) {
    c->tail = 0;
    c->nlight = 0;
    c->nchunk = 0;
    c->nheavy = 0;
    c->minrem = kInf;
    c->minsucc = kInf;
    c->theta = 0;
    c->fsize = 0;
    c->edges = 0;
    c->succ = 0;
    c->inserts = 0;
}

__device__ __forceinline__ Desc ld_desc(const Desc* p) {
    const uint4 v = __ldcg((const uint4*)p);
    Desc e;
    e.d = ((uint64_t)v.y << 32) | v.x;
    e.beg = (int32_t)v.z;
    e.len = (int32_t)v.w;
    return e;
}
__device__ __forceinline__ void st_desc(Desc* p, uint64_t d, int32_t beg, int32_t len) {
    __stcg((uint4*)p, make_uint4((uint32_t)d, (uint32_t)(d >> 32), (uint32_t)beg, (uint32_t)len));
}
__device__ __forceinline__ void st_desc_smem(Desc* p, uint64_t d, int32_t beg, int32_t len) {
    p->d = d;
    p->beg = beg;
    p->len = len;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Global warp rank, CTA-minor: consecutive work items land on different SMs, so a
// small round is spread over the whole GPU instead of the first few CTAs.
__device__ __forceinline__ int64_t warp_rank() { return (int64_t)(threadIdx.x >> 5) * gridDim.x + blockIdx.x; }

__host__ __device__ constexpr bool uses_min(int pol) { return pol == SSSP_DELTA || pol == SSSP_DIJKSTRA; }

// --------------------------------------------------------------------- per-warp staging
// Appends to the next queue, and light vertices waiting to be relaxed, are staged in a
// warp-private shared-memory buffer: one global atomicAdd per ~kQBuf appended ids
// instead of one per warp step, and the flush is a coalesced store.
constexpr int kWarps = kBlock / 32;
constexpr int kEnt = 4;     // queue entries per lane per Extract step
constexpr int kQBuf = 256;  // staged queue ids per warp (>= 32 * kArcs)
constexpr int kLBuf = 32 * kEnt + 32;  // staged light vertices per warp
static_assert(32 * kArcs <= kQBuf, "one relax step must fit the stage");

struct WarpStage {
    Desc light[kLBuf];
    int32_t q[kQBuf];
};

struct Acc {
    uint64_t minsucc = kInf;
    uint32_t succ = 0;
    uint32_t inserts = 0;
};

struct Warp {  // per-warp working state (qn, ln are warp-uniform)
    WarpStage* st;
    int32_t* qnext;
    RoundCnt* C;
    int32_t qn;
    int32_t ln;
    Acc acc;
};

__device__ __forceinline__ void wq_flush(Warp& W) {
    if (W.qn == 0) return;
    __syncwarp();
    int32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(&W.C->tail, W.qn);
    base = __shfl_sync(kFull, base, 0);
    for (int32_t i = lane_id(); i < W.qn; i += 32) W.qnext[base + i] = W.st->q[i];
    __syncwarp();
    W.qn = 0;
}

// stage the lanes' ids with pred (one id per lane)
__device__ __forceinline__ void wq_push1(Warp& W, bool pred, int32_t id) {
    const uint32_t mask = __ballot_sync(kFull, pred);
    if (!mask) return;
    const int32_t cnt = __popc(mask);
    if (W.qn + cnt > kQBuf) wq_flush(W);
    if (pred) W.st->q[W.qn + __popc(mask & lanemask_lt())] = id;
    W.qn += cnt;
}

// --------------------------------------------------------------------- relax
// WriteMin(delta[v], c) on the packed word, given a prior read `w`.
// Returns true iff this lane inserted v into Q (its flag bit was set) and must append it.
template <int POL, bool STATS>
__device__ __forceinline__ bool write_min(uint64_t* dist, int32_t v, uint64_t c, uint64_t w, Acc& acc) {
    while ((w & kVal) > c) {
        const uint64_t old = atomicCAS((unsigned long long*)(dist + v), (unsigned long long)w, (unsigned long long)c);
        if (old == w) {
            if (STATS) acc.succ++;
            if (uses_min(POL)) acc.minsucc = c < acc.minsucc ? c : acc.minsucc;
            return (w & kTop) != 0;
        }
        w = old;
    }
    return false;
}

// Relax kArcs arcs per lane (v < 0 = empty slot): filter loads, WriteMins, stage the
// inserted ids (Alg. 1 lines 5-6).
template <int POL, bool STATS>
__device__ __forceinline__ void relax_slots(const RunParams& p, const int32_t (&v)[kArcs], const uint64_t (&c)[kArcs],
                                            Warp& W) {
    uint64_t cur[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) cur[t] = v[t] >= 0 ? ld_cg_u64(p.dist + v[t]) : 0ull;
    int32_t cnt = 0;
    bool app[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) {
        app[t] = v[t] >= 0 && write_min<POL, STATS>(p.dist, v[t], c[t], cur[t], W.acc);
        cnt += app[t];
    }
    if (!__any_sync(kFull, cnt != 0)) return;
    const int32_t incl = warp_incl_scan(cnt);
    const int32_t tot = __shfl_sync(kFull, incl, 31);
    if (W.qn + tot > kQBuf) wq_flush(W);
    int32_t pos = W.qn + incl - cnt;
#pragma unroll
    for (int t = 0; t < kArcs; t++)
        if (app[t]) W.st->q[pos++] = v[t];
    W.qn += tot;
    if (STATS) W.acc.inserts += cnt;
}

// One chunk: arcs [beg, beg+len) of a vertex with key d, len <= kChunk.  Lane-strided
// so every load instruction of the warp reads 128 contiguous bytes.
template <int POL, bool STATS>
__device__ __forceinline__ void relax_chunk(const RunParams& p, uint64_t d, int32_t beg, int32_t len, Warp& W) {
    const int lane = lane_id();
    int32_t v[kArcs];
    uint64_t c[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) {
        const int32_t k = t * 32 + lane;
        v[t] = k < len ? ld_stream_i32(p.idx + beg + k) : -1;
        c[t] = d + (k < len ? ld_stream_u32(p.w + beg + k) : 0u);
    }
    relax_slots<POL, STATS>(p, v, c, W);
}

// Up to 32 vertices, one per lane (deg = 0 for none): the warp walks their
// concatenated arc lists; arc e belongs to the largest lane o with excl[o] <= e.
template <int POL, bool STATS>
__device__ __forceinline__ void relax_vertices(const RunParams& p, uint64_t d, int32_t beg, int32_t deg, Warp& W) {
    const int lane = lane_id();
    const int32_t incl = warp_incl_scan(deg);
    const int32_t total = __shfl_sync(kFull, incl, 31);
    const int32_t excl = incl - deg;
    const int32_t rowbase = beg - excl;  // CSR position of concatenated arc e of this lane = rowbase + e
    for (int32_t s0 = 0; s0 < total; s0 += 32 * kArcs) {
        int32_t v[kArcs];
        uint64_t c[kArcs];
#pragma unroll
        for (int t = 0; t < kArcs; t++) {
            const int32_t e = s0 + t * 32 + lane;
            int32_t o = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int32_t x = __shfl_sync(kFull, excl, o + step);
                if (x <= e) o += step;
            }
            const int32_t rb = __shfl_sync(kFull, rowbase, o);
            const uint64_t od = __shfl_sync(kFull, d, o);
            const bool ok = e < total;
            v[t] = ok ? ld_stream_i32(p.idx + rb + e) : -1;
            c[t] = od + (ok ? ld_stream_u32(p.w + rb + e) : 0u);
        }
        relax_slots<POL, STATS>(p, v, c, W);
    }
}

// Stage light vertices (live mode); light_relax_full relaxes them 32 at a time.
__device__ __forceinline__ void light_stage(bool pred, uint64_t d, int32_t beg, int32_t deg, Warp& W) {
    const uint32_t mask = __ballot_sync(kFull, pred);
    if (!mask) return;
    if (pred) st_desc_smem(&W.st->light[W.ln + __popc(mask & lanemask_lt())], d, beg, deg);
    W.ln += __popc(mask);
}

template <int POL, bool STATS>
__device__ __forceinline__ void light_relax_full(const RunParams& p, Warp& W) {
    const int lane = lane_id();
    int32_t done = 0;
    while (W.ln - done >= 32) {
        __syncwarp();
        const Desc e = W.st->light[done + lane];
        done += 32;
        relax_vertices<POL, STATS>(p, e.d, e.beg, e.len, W);
    }
    if (done) {  // move the remainder (< 32) to the front
        __syncwarp();
        const bool mv = lane < W.ln - done;
        Desc t;
        if (mv) t = W.st->light[done + lane];
        __syncwarp();
        if (mv) W.st->light[lane] = t;
        __syncwarp();
        W.ln -= done;
    }
}

template <int POL, bool STATS>
__device__ __forceinline__ void light_drain(const RunParams& p, Warp& W) {
    if (W.ln == 0) return;
    __syncwarp();
    const int lane = lane_id();
    Desc e;
    e.d = 0;
    e.beg = 0;
    e.len = 0;
    if (lane < W.ln) e = W.st->light[lane];
    __syncwarp();
    W.ln = 0;
    relax_vertices<POL, STATS>(p, e.d, e.beg, e.len, W);
}

// Cut the heavy lanes' vertices into kChunk-arc descriptors; one atomic per warp.
__device__ __forceinline__ void emit_chunks(const RunParams& p, bool heavy, uint64_t d, int32_t beg, int32_t deg,
                                            RoundCnt* C, bool stats) {
    const uint32_t hm = __ballot_sync(kFull, heavy);
    if (!hm) return;
    const int lane = lane_id();
    const int32_t nch = heavy ? (deg + kChunk - 1) / kChunk : 0;
    const int32_t incl = warp_incl_scan(nch);
    const int32_t tot = __shfl_sync(kFull, incl, 31);
    const int32_t excl = incl - nch;
    int32_t base = 0;
    if (lane == 0) {
        base = atomicAdd(&C->nchunk, tot);
        if (stats) atomicAdd(&C->nheavy, __popc(hm));
    }
    base = __shfl_sync(kFull, base, 0);
    for (int32_t j0 = 0; j0 < tot; j0 += 32) {
        const int32_t j = j0 + lane;
        int32_t o = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int32_t x = __shfl_sync(kFull, excl, o + step);
            if (x <= j) o += step;
        }
        const int32_t ob = __shfl_sync(kFull, beg, o);
        const int32_t oe = __shfl_sync(kFull, excl, o);
        const int32_t od = __shfl_sync(kFull, deg, o);
        const uint64_t odd = __shfl_sync(kFull, d, o);
        if (j < tot) {
            const int32_t k = (j - oe) * kChunk;
            st_desc(p.chunks + base + j, odd, ob + k, min(kChunk, od - k));
        }
    }
}

// --------------------------------------------------------------------- phase A
// Extract(theta): kEnt queue entries per lane per step, all loads issued together.
template <int POL, bool STATS, bool SNAP>
__device__ __forceinline__ void phase_a(const RunParams& p, const int32_t* __restrict__ qcur, int32_t q,
                                        uint64_t theta, Warp& W) {
    const int lane = lane_id();
    const int64_t gw = warp_rank();
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t minrem = kInf, fs = 0, edges = 0;
    // kEnt entries per lane only when every warp gets at least two such steps; small
    // queues are spread one entry per lane so that more warps share the round
    const int ent = (int64_t)q >= nwarps * (64 * kEnt) ? kEnt : 1;
    for (int64_t base = gw * (32 * ent); base < q; base += nwarps * (32 * ent)) {
        int32_t id[kEnt];
        uint64_t val[kEnt];
#pragma unroll
        for (int e = 0; e < kEnt; e++) {
            const int64_t i = base + e * 32 + lane;
            id[e] = (e < ent && i < q) ? ld_cg_i32(qcur + i) : -1;
        }
#pragma unroll
        for (int e = 0; e < kEnt; e++) val[e] = id[e] >= 0 ? (ld_cg_u64(p.dist + id[e]) & kVal) : kVal;
        int32_t beg[kEnt], deg[kEnt];
#pragma unroll
        for (int e = 0; e < kEnt; e++) {
            beg[e] = 0;
            deg[e] = 0;
            if (id[e] >= 0 && val[e] <= theta) {
                // delete u from Q; the returned word is u's key at deletion (<= val)
                val[e] = atomicOr((unsigned long long*)(p.dist + id[e]), (unsigned long long)kTop) & kVal;
                beg[e] = __ldg(p.off + id[e]);
                deg[e] = __ldg(p.off + id[e] + 1) - beg[e];
                if (p.ext_count) atomicAdd(p.ext_count + id[e], 1);
            } else if (id[e] >= 0) {
                deg[e] = -1;  // stays in Q
            }
        }
#pragma unroll
        for (int e = 0; e < kEnt; e++) {
            const bool rem = deg[e] < 0;
            const bool take = id[e] >= 0 && !rem;
            wq_push1(W, rem, id[e]);
            if (uses_min(POL) && rem) minrem = val[e] < minrem ? val[e] : minrem;
            if (STATS && take) {
                fs += 1;
                edges += (uint64_t)deg[e];
            }
            const bool heavy = take && deg[e] > kLight;
            const bool light = take && deg[e] > 0 && !heavy;
            emit_chunks(p, heavy, val[e], beg[e], deg[e], W.C, STATS);
            if (SNAP) {
                const int32_t ls = warp_append_slot(light, &W.C->nlight);
                if (light) st_desc(p.light + ls, val[e], beg[e], deg[e]);
            } else {
                light_stage(light, val[e], beg[e], deg[e], W);
            }
        }
        if (!SNAP) light_relax_full<POL, STATS>(p, W);
    }
    if (!SNAP) light_drain<POL, STATS>(p, W);
    if (uses_min(POL)) {
        minrem = warp_min_u64(minrem);
        if (lane == 0 && minrem != kInf) atomicMin(&W.C->minrem, (unsigned long long)minrem);
    }
    if (STATS) {
        fs = warp_sum(fs);
        edges = warp_sum(edges);
        if (lane == 0 && fs) atomicAdd(&W.C->fsize, (unsigned long long)fs);
        if (lane == 0 && edges) atomicAdd(&W.C->edges, (unsigned long long)edges);
    }
}

// --------------------------------------------------------------------- phase B
template <int POL, bool STATS, bool SNAP>
__device__ __forceinline__ void phase_b(const RunParams& p, int32_t nl, int32_t nc, Warp& W) {
    const int lane = lane_id();
    const int64_t gw = warp_rank();
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nb = SNAP ? ((int64_t)nl + 31) / 32 : 0;
    const int64_t total = nb + nc;
    int64_t item = gw;
    Desc nxt;
    if (item >= nb && item < total) nxt = ld_desc(p.chunks + (item - nb));
    for (; item < total; item += nwarps) {
        if (SNAP && item < nb) {
            const int64_t j = item * 32 + lane;
            Desc e;
            if (j < nl) {
                e = ld_desc(p.light + j);
            } else {
                e.d = 0;
                e.beg = 0;
                e.len = 0;
            }
            relax_vertices<POL, STATS>(p, e.d, e.beg, e.len, W);
            if (item + nwarps >= nb && item + nwarps < total) nxt = ld_desc(p.chunks + (item + nwarps - nb));
        } else {
            const Desc e = nxt;
            if (item + nwarps < total) nxt = ld_desc(p.chunks + (item + nwarps - nb));  // prefetch
            relax_chunk<POL, STATS>(p, e.d, e.beg, e.len, W);
        }
    }
}

template <int POL, bool STATS>
__device__ __forceinline__ void flush_acc(Warp& W) {
    wq_flush(W);
    if (uses_min(POL)) {
        const uint64_t mn = warp_min_u64(W.acc.minsucc);
        if (lane_id() == 0 && mn != kInf) atomicMin(&W.C->minsucc, (unsigned long long)mn);
    }
    if (STATS) {
        const uint32_t s = warp_sum(W.acc.succ), ins = warp_sum(W.acc.inserts);
        if (lane_id() == 0 && s) atomicAdd(&W.C->succ, (unsigned long long)s);
        if (lane_id() == 0 && ins) atomicAdd(&W.C->inserts, (unsigned long long)ins);
    }
    W.acc = Acc();
}

// --------------------------------------------------------------------- ExtDist for rho
struct SmemKey {
    const uint64_t* a;
    __device__ uint64_t operator()(int64_t i) const { return a[i]; }
};
struct QueueVal {  // value of the i-th queued id (flag bit masked off), read through L2
    const int32_t* queue;
    const uint64_t* dist;
    __device__ uint64_t operator()(int64_t i) const { return ld_cg_u64(dist + ld_cg_i32(queue + i)) & kVal; }
};

__device__ __forceinline__ uint64_t sample_index(uint64_t seed, int64_t round, uint64_t j, uint64_t q) {
    return splitmix64(seed ^ splitmix64(((uint64_t)round << 32) | j)) % q;
}

// k-th smallest (1-based) of s <= blockDim keys in shared memory by rank counting:
// the key x with #{< x} < k <= #{<= x}.  One pass of broadcast reads, two barriers.
__device__ __forceinline__ uint64_t cta_kth_by_rank(const uint64_t* keys, int s, uint64_t k, SelectSmem& sm) {
    const int tid = threadIdx.x;
    if (tid < s) {
        const uint64_t x = keys[tid];
        uint32_t lt = 0, le = 0;
        for (int j = 0; j < s; j++) {
            const uint64_t y = keys[j];
            lt += y < x;
            le += y <= x;
        }
        if (lt < k && k <= le) sm.bcast[0] = x;  // every writer writes the same value
    }
    __syncthreads();
    const uint64_t th = sm.bcast[0];
    __syncthreads();
    return th;
}

// --------------------------------------------------------------------- the round loop
template <int POL, bool STATS, bool SNAP>
__global__ void __launch_bounds__(kBlock, kMinBlocks) sssp_round_loop(RunParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpStage* stage = (WarpStage*)smem_raw;                            // [kWarps]
    uint64_t* s_keys = (uint64_t*)(smem_raw + kWarps * sizeof(WarpStage)); // [kSmemSamples]
    SelectSmem& sm = *(SelectSmem*)(s_keys + kSmemSamples);
    Ctrl* ctrl = p.ctrl;
    Warp W;
    W.st = stage + (threadIdx.x >> 5);
    W.qn = 0;
    W.ln = 0;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;

    // Alg. 1 lines 1-2: delta[.] = +inf (not in Q), delta[s] = 0 (in Q), queue = {s}
    for (int64_t i = gtid; i < p.n; i += gsize) p.dist[i] = (i == p.source) ? 0ull : kInf;
    if (p.ext_count)
        for (int64_t i = gtid; i < p.n; i += gsize) p.ext_count[i] = 0;
    if (gtid == 0) {
        p.q0[0] = p.source;
        for (int c = 0; c < 3; c++) reset_cnt(&ctrl->cnt[c]);
        ctrl->cnt[0].tail = 1;    // |Q_1| = 1
        ctrl->cnt[0].minrem = 0;  // min_Q delta = delta[s] = 0
        ctrl->status = 0;
        ctrl->rounds = 0;
        ctrl->tot_extracted = ctrl->tot_edges = ctrl->tot_succ = ctrl->tot_inserts = 0;
        ctrl->tot_qscan = ctrl->max_q = ctrl->max_f = 0;
    }
    grid_sync(&ctrl->bar);

    uint64_t theta_prev = 0;
    int warm = 0;
    int64_t r = 1;
    for (;; r++) {
        RoundCnt* P = &ctrl->cnt[(r + 2) % 3];
        RoundCnt* C = &ctrl->cnt[r % 3];
        const int32_t q = ld_volatile_i32(&P->tail);  // |Q_r|
        if (q == 0) break;                             // while |Q| > 0
        if (r > p.max_rounds) {
            if (gtid == 0) ctrl->status = SSSP_ERR_ROUNDS;
            break;
        }
        uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
        if (STATS && gtid == 0) t0 = globaltimer();
        if (gtid == 0) reset_cnt(&ctrl->cnt[(r + 1) % 3]);
        const int32_t* qcur = (r & 1) ? p.q0 : p.q1;
        int32_t* qnext = (r & 1) ? p.q1 : p.q0;

        // ---- ExtDist (Table tab:framework)
        uint64_t theta;
        if (POL == SSSP_BELLMAN_FORD) {
            theta = kInf;
        } else if (POL == SSSP_DIJKSTRA || POL == SSSP_DELTA) {
            const uint64_t a = ld_volatile_u64((const uint64_t*)&P->minrem);
            const uint64_t b = ld_volatile_u64((const uint64_t*)&P->minsucc);
            const uint64_t minq = a < b ? a : b;  // <= min_{v in Q} delta[v] (exact in snapshot mode)
            if (POL == SSSP_DIJKSTRA) {
                theta = minq;
            } else {
                const uint64_t D = p.param;  // theta_i = i*Delta, skipping empty steps (reading R2)
                const uint64_t x = theta_prev > kInf - D ? kInf : theta_prev + D;
                const uint64_t y = (minq / D + (minq % D != 0)) * D;
                theta = x > y ? x : y;
                theta_prev = theta;
            }
        } else {  // rho
            uint64_t rho = p.param;
            if (!(p.flags & SSSP_RUN_NO_WARMUP) && (uint64_t)q > rho && warm < 2) {
                warm++;
                rho = rho / 10 ? rho / 10 : 1;  // reading R7
            }
            const uint64_t s = sample_count((uint64_t)q, rho);
            if ((uint64_t)q <= rho) {
                theta = kInf;  // |Q| <= rho: extract all
            } else if (!(p.flags & SSSP_RUN_RHO_EXACT) && s <= (uint64_t)kSmemSamples) {
                // every CTA draws the same samples and selects the same theta: no barrier
                for (uint64_t j = threadIdx.x; j < s; j += blockDim.x)
                    s_keys[j] = ld_cg_u64(p.dist + ld_cg_i32(qcur + sample_index(p.seed, r, j, (uint64_t)q))) & kVal;
                __syncthreads();
                uint64_t k = (rho * s + (uint64_t)q - 1) / (uint64_t)q;
                k = k < 1 ? 1 : (k > s ? s : k);
                theta = s <= (uint64_t)kRankSelect ? cta_kth_by_rank(s_keys, (int)s, k, sm)
                                                   : cta_kth_smallest(SmemKey{s_keys}, (int64_t)s, k, sm);
            } else {
                if (blockIdx.x == 0) {
                    uint64_t th;
                    if (p.flags & SSSP_RUN_RHO_EXACT) {
                        th = cta_kth_smallest(QueueVal{qcur, p.dist}, q, rho, sm);
                    } else {
                        for (uint64_t j = threadIdx.x; j < s; j += blockDim.x)
                            p.samples[j] =
                                ld_cg_u64(p.dist + ld_cg_i32(qcur + sample_index(p.seed, r, j, (uint64_t)q))) & kVal;
                        __syncthreads();
                        uint64_t k = (rho * s + (uint64_t)q - 1) / (uint64_t)q;
                        k = k < 1 ? 1 : (k > s ? s : k);
                        th = cta_kth_smallest(ArrayKey{p.samples}, (int64_t)s, k, sm);
                    }
                    if (threadIdx.x == 0) C->theta = th;
                }
                grid_sync(&ctrl->bar);
                theta = ld_volatile_u64((const uint64_t*)&C->theta);
            }
        }
        if (STATS && gtid == 0) t1 = globaltimer();

        // ---- phase A: Extract(theta) (+ light relax in live mode)
        W.qnext = qnext;
        W.C = C;
        phase_a<POL, STATS, SNAP>(p, qcur, q, theta, W);
        flush_acc<POL, STATS>(W);
        grid_sync(&ctrl->bar);
        if (STATS && gtid == 0) t2 = globaltimer();
        // ---- phase B: heavy chunks (+ light list in snapshot mode)
        const int32_t nc = ld_volatile_i32(&C->nchunk);
        const int32_t nl = SNAP ? ld_volatile_i32(&C->nlight) : 0;
        if (nc + nl > 0) {
            phase_b<POL, STATS, SNAP>(p, nl, nc, W);
            flush_acc<POL, STATS>(W);
            grid_sync(&ctrl->bar);
        }
        if (STATS && gtid == 0) t3 = globaltimer();

        if (STATS && gtid == 0) {
            const int64_t f = (int64_t)C->fsize;
            if (p.trace && r - 1 < p.trace_cap) {
                sssp_round* t = p.trace + (r - 1);
                t->qsize = q;
                t->fsize = f;
                t->edges = (int64_t)C->edges;
                t->inserts = (int64_t)C->inserts;
                t->succ = (int64_t)C->succ;
                t->theta = theta;
                t->nheavy = (int64_t)C->nheavy;
                t->t_theta_ns = (int64_t)(t1 - t0);
                t->t_extract_ns = (int64_t)(t2 - t1);
                t->t_relax_ns = (int64_t)(t3 - t2);
                t->reserved0 = C->nchunk;
                t->reserved1 = 0;
            }
            ctrl->tot_extracted += f;
            ctrl->tot_edges += (int64_t)C->edges;
            ctrl->tot_succ += (int64_t)C->succ;
            ctrl->tot_inserts += (int64_t)C->inserts;
            ctrl->tot_qscan += q;
            ctrl->max_q = q > ctrl->max_q ? q : ctrl->max_q;
            ctrl->max_f = f > ctrl->max_f ? f : ctrl->max_f;
        }
    }
    if (gtid == 0) ctrl->rounds = r - 1;
    // S6 output: strip the flag bit (every reached vertex was extracted; INF stays INF)
    for (int64_t i = gtid; i < p.n; i += gsize) {
        const uint64_t x = __ldcg((const unsigned long long*)(p.dist + i));
        if (x != kInf && (x & kTop)) p.dist[i] = x & kVal;
    }
}

// --------------------------------------------------------------------- CSR validation
__global__ void validate_csr(int32_t n, int64_t m, const int32_t* off, const int32_t* idx, const uint32_t* w,
                             int32_t* err) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    if (gtid == 0 && (off[0] != 0 || (int64_t)off[n] != m)) atomicOr(err, 1);
    for (int64_t i = gtid; i < n; i += gsize)
        if (off[i] > off[i + 1]) atomicOr(err, 2);
    for (int64_t e = gtid; e < m; e += gsize) {
        if (idx[e] < 0 || idx[e] >= n) atomicOr(err, 4);
        if (w[e] < 1) atomicOr(err, 8);
    }
}

}  // namespace sssp

// ======================================================================= host API
using namespace sssp;

struct sssp_handle {
    int32_t n;
    int64_t m;
    const int32_t* off;
    const int32_t* idx;
    const uint32_t* w;
    cudaStream_t stream;
    uint32_t flags;
    RunParams base;  // carved workspace pointers
    uint64_t* ws_dist;
    Ctrl* ctrl;
    Ctrl* h_ctrl;  // pinned host mirror for result readback
    int device;
    cudaEvent_t ev[2];
    int num_sms;
    int grid[4][2][2];
};

namespace {

struct Layout {
    uint64_t* dist;
    int32_t *q0, *q1;
    Desc *light, *chunks;
    uint64_t* samples;
    Ctrl* ctrl;
    int32_t* err;
    size_t bytes;
};

Layout carve(void* base, int32_t n, int64_t m) {
    Carver c(base);
    Layout L;
    // chunks per round <= sum over heavy extracted vertices of ceil(deg/kChunk)
    const int64_t ccap = m / kChunk + std::min<int64_t>(n, m / (kLight + 1)) + 1;
    L.ctrl = c.take<Ctrl>(1);
    L.err = c.take<int32_t>(32);
    L.dist = c.take<uint64_t>(n);
    L.q0 = c.take<int32_t>(n);
    L.q1 = c.take<int32_t>(n);
    L.light = c.take<Desc>(n);
    L.chunks = c.take<Desc>(ccap);
    L.samples = c.take<uint64_t>(kMaxSamples);
    L.bytes = align_up(c.off, 256);
    return L;
}

typedef void (*KernelFn)(RunParams);

constexpr size_t kSmemBytes = kWarps * sizeof(WarpStage) + kSmemSamples * sizeof(uint64_t) + sizeof(SelectSmem);

template <int POL>
KernelFn kernel_for_pol(bool stats, bool snap) {
    if (stats) return snap ? sssp_round_loop<POL, true, true> : sssp_round_loop<POL, true, false>;
    return snap ? sssp_round_loop<POL, false, true> : sssp_round_loop<POL, false, false>;
}

KernelFn kernel_for(int pol, bool stats, bool snap) {
    switch (pol) {
        case SSSP_RHO: return kernel_for_pol<SSSP_RHO>(stats, snap);
        case SSSP_DELTA: return kernel_for_pol<SSSP_DELTA>(stats, snap);
        case SSSP_BELLMAN_FORD: return kernel_for_pol<SSSP_BELLMAN_FORD>(stats, snap);
        case SSSP_DIJKSTRA: return kernel_for_pol<SSSP_DIJKSTRA>(stats, snap);
    }
    return nullptr;
}

}  // namespace

extern "C" {

size_t sssp_workspace_bytes(int32_t n, int64_t m, uint32_t flags) {
    (void)flags;
    if (n < 1 || n > 2147483646 || m < 0 || m > 2147483647LL) return 0;
    return carve(nullptr, n, m).bytes;
}

sssp_status sssp_create(int32_t n, int64_t m, const int32_t* d_offsets, const int32_t* d_indices,
                        const uint32_t* d_weights, void* d_workspace, size_t ws_bytes, sssp_stream_t stream,
                        uint32_t flags, sssp_handle** out) {
    if (!out) return set_error(SSSP_ERR_INVALID, "sssp_create: out is NULL");
    *out = nullptr;
    if (n < 1 || n > 2147483646) return set_error(SSSP_ERR_INVALID, "sssp_create: n=%d outside [1, 2^31-2]", n);
    if (m < 0 || m > 2147483647LL) return set_error(SSSP_ERR_INVALID, "sssp_create: m=%lld outside [0, 2^31-1]", (long long)m);
    if (!d_offsets || (m > 0 && (!d_indices || !d_weights)) || !d_workspace)
        return set_error(SSSP_ERR_INVALID, "sssp_create: NULL graph or workspace pointer");
    if ((uintptr_t)d_workspace % 256) return set_error(SSSP_ERR_INVALID, "sssp_create: workspace not 256-byte aligned");
    const size_t need = sssp_workspace_bytes(n, m, flags);
    if (ws_bytes < need)
        return set_error(SSSP_ERR_INVALID, "sssp_create: workspace %zu bytes < required %zu", ws_bytes, need);
    int dev = 0;
    cudaError_t e = bind_device_of(d_workspace, &dev);
    if (e != cudaSuccess) return cuda_error(e, "sssp_create: workspace is not device memory");
    int major = 0, coop = 0, sms = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (major != 10 || !coop)
        return set_error(SSSP_ERR_DEVICE, "sssp_create: needs an sm_100 device with cooperative launch (cc major %d)", major);

    Layout L = carve(d_workspace, n, m);
    sssp_handle* h = new sssp_handle();
    h->n = n;
    h->m = m;
    h->off = d_offsets;
    h->idx = d_indices;
    h->w = d_weights;
    h->stream = (cudaStream_t)stream;
    h->flags = flags;
    h->device = dev;
    h->num_sms = sms;
    h->ws_dist = L.dist;
    h->ctrl = L.ctrl;
    RunParams& b = h->base;
    memset(&b, 0, sizeof(b));
    b.n = n;
    b.m = m;
    b.off = d_offsets;
    b.idx = d_indices;
    b.w = d_weights;
    b.q0 = L.q0;
    b.q1 = L.q1;
    b.light = L.light;
    b.chunks = L.chunks;
    b.samples = L.samples;
    b.ctrl = L.ctrl;
    for (int pol = 0; pol < 4; pol++)
        for (int st = 0; st < 2; st++)
            for (int sn = 0; sn < 2; sn++) {
                int per_sm = 0;
                e = cudaFuncSetAttribute((const void*)kernel_for(pol, st, sn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kernel_for(pol, st, sn),
                                                                      kBlock, kSmemBytes);
                if (e != cudaSuccess || per_sm < 1) {
                    delete h;
                    return e != cudaSuccess ? cuda_error(e, "occupancy query")
                                            : set_error(SSSP_ERR_DEVICE, "round-loop kernel cannot be resident");
                }
                h->grid[pol][st][sn] = per_sm * sms;
            }
    e = cudaMallocHost((void**)&h->h_ctrl, sizeof(Ctrl));
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev[0]);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev[1]);
    if (e != cudaSuccess) {
        delete h;
        return cuda_error(e, "sssp_create: host resources");
    }
    // the barrier counter must start at a multiple of 2^31; the rest is reset per run
    e = cudaMemsetAsync(L.ctrl, 0, sizeof(Ctrl), h->stream);
    if (e == cudaSuccess && (flags & SSSP_VALIDATE)) {
        cudaMemsetAsync(L.err, 0, sizeof(int32_t), h->stream);
        validate_csr<<<sms * 4, 256, 0, h->stream>>>(n, m, d_offsets, d_indices, d_weights, L.err);
        e = cudaGetLastError();
        int32_t herr = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, L.err, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess && herr) {
            cudaFreeHost(h->h_ctrl);
            delete h;
            return set_error(SSSP_ERR_INVALID_GRAPH, "sssp_create: invalid CSR (%s%s%s%s)",
                             (herr & 1) ? "offsets[0]!=0 or offsets[n]!=m " : "", (herr & 2) ? "offsets decrease " : "",
                             (herr & 4) ? "index out of range " : "", (herr & 8) ? "weight < 1" : "");
        }
    }
    if (e != cudaSuccess) {
        cudaFreeHost(h->h_ctrl);
        delete h;
        return cuda_error(e, "sssp_create");
    }
    *out = h;
    return SSSP_OK;
}

sssp_status sssp_run_ex(sssp_handle* h, int32_t source, sssp_policy policy, uint64_t param,
                        const sssp_run_opts* opts, uint64_t* d_dist_out, sssp_run_stats* stats) {
    if (!h) return set_error(SSSP_ERR_INVALID, "sssp_run: NULL handle");
    if (!d_dist_out) return set_error(SSSP_ERR_INVALID, "sssp_run: NULL d_dist_out");
    if (source < 0 || source >= h->n) return set_error(SSSP_ERR_RANGE, "sssp_run: source %d outside [0, %d)", source, h->n);
    if (policy < SSSP_RHO || policy > SSSP_DIJKSTRA) return set_error(SSSP_ERR_INVALID, "sssp_run: unknown policy %d", (int)policy);
    if ((policy == SSSP_RHO || policy == SSSP_DELTA) && param == 0)
        return set_error(SSSP_ERR_INVALID, "sssp_run: param (rho / Delta) must be >= 1");
    cudaError_t de = cudaSetDevice(h->device);
    if (de != cudaSuccess) return cuda_error(de, "cudaSetDevice");
    sssp_run_opts o;
    memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    const bool st = (o.flags & SSSP_RUN_STATS) != 0;
    const bool sn = (o.flags & SSSP_RUN_SNAPSHOT) != 0;
    RunParams p = h->base;
    p.dist = d_dist_out;
    p.source = source;
    p.param = param;
    p.flags = o.flags;
    p.seed = o.seed;
    p.max_rounds = o.max_rounds > 0 ? o.max_rounds : 4 * (int64_t)h->n + 64;
    p.trace = st ? (sssp_round*)o.d_trace : nullptr;
    p.trace_cap = o.trace_cap;
    p.ext_count = o.d_ext_count;
    KernelFn k = kernel_for(policy, st, sn);
    const int grid = h->grid[policy][st][sn];
    void* args[] = {&p};
    cudaEventRecord(h->ev[0], h->stream);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kBlock), args, kSmemBytes, h->stream);
    if (e != cudaSuccess) return cuda_error(e, "round-loop launch");
    cudaEventRecord(h->ev[1], h->stream);
    e = cudaMemcpyAsync(&h->h_ctrl->status, &h->ctrl->status, sizeof(Ctrl) - offsetof(Ctrl, status),
                        cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_error(e, "round loop");
    const Ctrl* c = h->h_ctrl;
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->rounds = c->rounds;
        stats->extracted = c->tot_extracted;
        stats->edges = c->tot_edges;
        stats->succ = c->tot_succ;
        stats->inserts = c->tot_inserts;
        stats->queue_scanned = c->tot_qscan;
        stats->max_queue = c->max_q;
        stats->max_frontier = c->max_f;
        stats->grid_blocks = grid;
        stats->block_threads = kBlock;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
        stats->kernel_ms = ms;
    }
    if (c->status == SSSP_ERR_ROUNDS)
        return set_error(SSSP_ERR_ROUNDS, "sssp_run: exceeded max_rounds=%lld", (long long)p.max_rounds);
    return SSSP_OK;
}

sssp_status sssp_run(sssp_handle* h, int32_t source, sssp_policy policy, uint64_t param, uint64_t* d_dist_out,
                     sssp_run_stats* stats) {
    return sssp_run_ex(h, source, policy, param, nullptr, d_dist_out, stats);
}

sssp_status sssp_run_host(sssp_handle* h, int32_t source, sssp_policy policy, uint64_t param, uint64_t* h_dist_out,
                          sssp_run_stats* stats) {
    if (!h) return set_error(SSSP_ERR_INVALID, "sssp_run_host: NULL handle");
    if (!h_dist_out) return set_error(SSSP_ERR_INVALID, "sssp_run_host: NULL h_dist_out");
    sssp_status s = sssp_run_ex(h, source, policy, param, nullptr, h->ws_dist, stats);
    if (s != SSSP_OK) return s;
    cudaError_t e = cudaMemcpyAsync(h_dist_out, h->ws_dist, (size_t)h->n * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_error(e, "sssp_run_host copy-out");
    return SSSP_OK;
}

sssp_status sssp_destroy(sssp_handle* h) {
    if (!h) return SSSP_OK;
    if (h->h_ctrl) cudaFreeHost(h->h_ctrl);
    if (h->ev[0]) cudaEventDestroy(h->ev[0]);
    if (h->ev[1]) cudaEventDestroy(h->ev[1]);
    delete h;
    return SSSP_OK;
}

}  // extern "C"
