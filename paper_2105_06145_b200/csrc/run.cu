// run.cu — the stepping-algorithm round loop (Alg. 1) as ONE persistent
// cooperative kernel, plus the sssp_* handle API.
//
// Per round r:
//   ExtDist   theta_r per policy (Table tab:framework).  BF / Delta* /
//             Dijkstra: a scalar every CTA derives identically; rho: CTA 0 samples
//             the queue and radix-selects, then one grid barrier.
//   Extract   (array LaB-PQ P:1011-1012) one pass over the compacted
//             queue: ids with delta <= theta have their flag cleared and go to the
//             frontier with a snapshot of delta (reading R8), binned by degree
//             into light entries and heavy chunks; the rest are compacted into the
//             next queue.  Warp ballots + one atomic per warp.        grid barrier
//   Relax     (Alg. 1 lines 4-6) warps pull work items (32 light
//             vertices, or one 256-arc chunk of a heavy vertex) from an atomic
//             counter; per arc: plain L2 load filter, WriteMin = atomicMin.u64
//             (P:697), on success Update(v) = atomicOr on the flag bitmap, and
//             the 0->1 winner appends v to the next queue.         grid barrier
//   loop while |Q| > 0: |Q_{r+1}| is the next queue's tail counter.
#include <stdio.h>

#include <algorithm>
#include <string.h>

#include "common.cuh"
#include "internal.h"

namespace sssp {

constexpr int kLightMax = 64;  // out-degree <= kLightMax: relaxed in warp batches of 32 vertices
constexpr int kChunk = 256;    // heavy vertices are split into chunks of kChunk arcs
constexpr int kBlock = 512;    // threads per CTA of the round loop
constexpr int kUnroll = 4;     // arcs per lane in flight

// A frontier entry: the extracted vertex's snapshot key and its CSR row.
struct __align__(16) FEntry {
    uint64_t d;
    int32_t beg;
    int32_t deg;
};

struct __align__(128) RoundCnt {
    int32_t tail;   // next-queue write cursor (remaining ids, then appended ids)
    int32_t nlight; // light frontier entries
    int32_t work;   // relax work-item counter
    int32_t pad0;
    unsigned long long heavy_pack;  // (#heavy << 32) | #chunks
    unsigned long long minrem;      // min key among ids kept in Q by Extract
    unsigned long long minsucc;     // min successful WriteMin value
    unsigned long long theta;
    unsigned long long edges;       // STATS
    unsigned long long succ;        // STATS
    unsigned long long inserts;     // STATS
    unsigned long long pad1[6];
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
    uint32_t* bm;
    int32_t* q0;
    int32_t* q1;
    FEntry* light;
    FEntry* heavy;
    int32_t* heavy_cb;
    int32_t* chunk_owner;
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
    c->work = 0;
    c->heavy_pack = 0;
    c->minrem = kInf;
    c->minsucc = kInf;
    c->theta = 0;
    c->edges = 0;
    c->succ = 0;
    c->inserts = 0;
}

__device__ __forceinline__ FEntry ld_entry(const FEntry* p) {
    uint4 v = __ldcg((const uint4*)p);
    FEntry e;
    e.d = ((uint64_t)v.y << 32) | v.x;
    e.beg = (int32_t)v.z;
    e.deg = (int32_t)v.w;
    return e;
}
__device__ __forceinline__ void st_entry(FEntry* p, uint64_t d, int32_t beg, int32_t deg) {
    uint4 v = make_uint4((uint32_t)d, (uint32_t)(d >> 32), (uint32_t)beg, (uint32_t)deg);
    __stcg((uint4*)p, v);
}

__host__ __device__ constexpr bool uses_min(int pol) { return pol == SSSP_DELTA || pol == SSSP_DIJKSTRA; }

// --------------------------------------------------------------------- Extract
template <int POL, bool STATS>
__device__ __forceinline__ void extract_phase(const RunParams& p, const int32_t* __restrict__ qcur,
                                              int32_t* __restrict__ qnext, int32_t q, uint64_t theta, RoundCnt* C) {
    const int lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t minrem = kInf;
    uint64_t edges = 0;
    for (int64_t base = gw * 32; base < q; base += nwarps * 32) {
        const int64_t i = base + lane;
        const bool valid = i < q;
        const int32_t id = valid ? ld_cg_i32(qcur + i) : 0;
        const uint64_t d = valid ? ld_cg_u64(p.dist + id) : kInf;
        const bool take = valid && d <= theta;
        const bool rem = valid && !take;
        int32_t beg = 0, deg = 0;
        if (take) {
            beg = __ldg(p.off + id);
            deg = __ldg(p.off + id + 1) - beg;
            atomicAnd(p.bm + (id >> 5), ~(1u << (id & 31)));  // delete from Q
            if (p.ext_count) atomicAdd(p.ext_count + id, 1);
        }
        // ids that stay in Q are compacted into the next queue
        const int32_t rs = warp_append_slot(rem, &C->tail);
        if (rem) qnext[rs] = id;
        if (uses_min(POL) && rem) minrem = d < minrem ? d : minrem;
        // light frontier entries
        const bool heavy = take && deg > kLightMax;
        const bool light = take && !heavy;
        const int32_t ls = warp_append_slot(light, &C->nlight);
        if (light) st_entry(p.light + ls, d, beg, deg);
        // heavy vertices: one packed atomic gives (slot, first chunk) consistently
        const uint32_t hm = __ballot_sync(kFull, heavy);
        if (hm) {
            const int32_t nch = heavy ? (deg + kChunk - 1) / kChunk : 0;
            const int32_t incl = warp_incl_scan(nch);
            const int32_t tot = __shfl_sync(kFull, incl, 31);
            unsigned long long old = 0;
            if (lane == 0) old = atomicAdd(&C->heavy_pack, ((unsigned long long)__popc(hm) << 32) | (unsigned)tot);
            old = __shfl_sync(kFull, old, 0);
            if (heavy) {
                const int32_t slot = (int32_t)(old >> 32) + __popc(hm & lanemask_lt());
                const int32_t cb = (int32_t)(old & 0xFFFFFFFFu) + incl - nch;
                st_entry(p.heavy + slot, d, beg, deg);
                __stcg(p.heavy_cb + slot, cb);
                for (int32_t j = 0; j < nch; j++) __stcg(p.chunk_owner + cb + j, slot);
            }
        }
        if (STATS && take) edges += (uint64_t)deg;
    }
    if (uses_min(POL)) {
        minrem = warp_min_u64(minrem);
        if (lane == 0 && minrem != kInf) atomicMin(&C->minrem, (unsigned long long)minrem);
    }
    if (STATS) {
        edges = warp_sum(edges);
        if (lane == 0 && edges) atomicAdd(&C->edges, (unsigned long long)edges);
    }
}

// --------------------------------------------------------------------- Relax
struct RelaxAcc {
    uint64_t minsucc = kInf;
    uint64_t succ = 0;
    uint64_t inserts = 0;
};

// WriteMin(delta[v], c) and, on success, Q.Update(v) (Alg. 1 lines 5-6).
// Returns true iff this lane must append v to the queue (its flag went 0 -> 1).
template <int POL, bool STATS>
__device__ __forceinline__ bool relax_arc(const RunParams& p, int32_t v, uint64_t c, RelaxAcc& acc) {
    if (c < ld_cg_u64(p.dist + v)) {  // plain-load filter: most candidates lose
        const uint64_t old = atomic_min_u64(p.dist + v, c);
        if (c < old) {
            if (STATS) acc.succ++;
            if (uses_min(POL)) acc.minsucc = c < acc.minsucc ? c : acc.minsucc;
            const uint32_t bit = 1u << (v & 31);
            return !(atomicOr(p.bm + (v >> 5), bit) & bit);
        }
    }
    return false;
}

// Append the lanes' flagged ids (up to kUnroll per lane) with one atomic per warp.
__device__ __forceinline__ void warp_append_many(const int32_t (&v)[kUnroll], const bool (&app)[kUnroll],
                                                 int32_t* cursor, int32_t* out, RelaxAcc& acc, bool stats) {
    int32_t cnt = 0;
#pragma unroll
    for (int t = 0; t < kUnroll; t++) cnt += app[t];
    const uint32_t any = __ballot_sync(kFull, cnt != 0);
    if (!any) return;
    const int32_t incl = warp_incl_scan(cnt);
    const int32_t tot = __shfl_sync(kFull, incl, 31);
    int32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(cursor, tot);
    base = __shfl_sync(kFull, base, 0);
    int32_t pos = base + incl - cnt;
#pragma unroll
    for (int t = 0; t < kUnroll; t++)
        if (app[t]) out[pos++] = v[t];
    if (stats) acc.inserts += cnt;
}

// Arcs [b, e) of one vertex with snapshot key d, all lanes of the warp.
template <int POL, bool STATS>
__device__ __forceinline__ void relax_row(const RunParams& p, uint64_t d, int32_t b, int32_t e, int32_t* qnext,
                                          RoundCnt* C, RelaxAcc& acc) {
    const int lane = lane_id();
    for (int32_t base = b; base < e; base += 32 * kUnroll) {
        int32_t v[kUnroll];
        uint32_t wt[kUnroll];
        bool app[kUnroll];
#pragma unroll
        for (int t = 0; t < kUnroll; t++) {
            const int32_t k = base + t * 32 + lane;
            v[t] = k < e ? ld_stream_i32(p.idx + k) : -1;
            wt[t] = k < e ? ld_stream_u32(p.w + k) : 0u;
        }
#pragma unroll
        for (int t = 0; t < kUnroll; t++) app[t] = v[t] >= 0 && relax_arc<POL, STATS>(p, v[t], d + wt[t], acc);
        warp_append_many(v, app, &C->tail, qnext, acc, STATS);
    }
}

// 32 light frontier entries: the warp walks their concatenated arc lists.
template <int POL, bool STATS>
__device__ __forceinline__ void relax_light_batch(const RunParams& p, int32_t batch, int32_t nl, int32_t* qnext,
                                                  RoundCnt* C, RelaxAcc& acc) {
    const int lane = lane_id();
    const int32_t j = batch * 32 + lane;
    FEntry me;
    if (j < nl) {
        me = ld_entry(p.light + j);
    } else {
        me.d = 0;
        me.beg = 0;
        me.deg = 0;
    }
    const int32_t incl = warp_incl_scan(me.deg);
    const int32_t total = __shfl_sync(kFull, incl, 31);
    const int32_t excl = incl - me.deg;
    for (int32_t base = 0; base < total; base += 32 * kUnroll) {
        int32_t v[kUnroll];
        uint32_t wt[kUnroll];
        uint64_t dd[kUnroll];
        bool app[kUnroll];
#pragma unroll
        for (int t = 0; t < kUnroll; t++) {
            const int32_t eidx = base + t * 32 + lane;
            // owner = largest lane o with excl[o] <= eidx (binary search over lanes)
            int32_t o = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int32_t x = __shfl_sync(kFull, excl, o + step);
                if (x <= eidx) o += step;
            }
            const int32_t ob = __shfl_sync(kFull, me.beg, o);
            const int32_t oe = __shfl_sync(kFull, excl, o);
            dd[t] = __shfl_sync(kFull, me.d, o);
            const bool ok = eidx < total;
            const int32_t k = ob + (eidx - oe);
            v[t] = ok ? ld_stream_i32(p.idx + k) : -1;
            wt[t] = ok ? ld_stream_u32(p.w + k) : 0u;
        }
#pragma unroll
        for (int t = 0; t < kUnroll; t++) app[t] = v[t] >= 0 && relax_arc<POL, STATS>(p, v[t], dd[t] + wt[t], acc);
        warp_append_many(v, app, &C->tail, qnext, acc, STATS);
    }
}

template <int POL, bool STATS>
__device__ __forceinline__ void relax_phase(const RunParams& p, int32_t* __restrict__ qnext, RoundCnt* C) {
    const int lane = lane_id();
    const int32_t nl = ld_volatile_i32(&C->nlight);
    const unsigned long long hp = ld_volatile_u64((const uint64_t*)&C->heavy_pack);
    const int32_t nchunks = (int32_t)(hp & 0xFFFFFFFFull);
    const int32_t nbatch = (nl + 31) / 32;
    const int32_t total = nbatch + nchunks;
    RelaxAcc acc;
    for (;;) {
        int32_t item = 0;
        if (lane == 0) item = atomicAdd(&C->work, 1);
        item = __shfl_sync(kFull, item, 0);
        if (item >= total) break;
        if (item < nbatch) {
            relax_light_batch<POL, STATS>(p, item, nl, qnext, C, acc);
        } else {
            const int32_t c = item - nbatch;
            const int32_t o = ld_cg_i32(p.chunk_owner + c);
            const FEntry e = ld_entry(p.heavy + o);
            const int32_t start = (c - ld_cg_i32(p.heavy_cb + o)) * kChunk;
            const int32_t end = min(start + kChunk, e.deg);
            relax_row<POL, STATS>(p, e.d, e.beg + start, e.beg + end, qnext, C, acc);
        }
    }
    if (uses_min(POL)) {
        const uint64_t m = warp_min_u64(acc.minsucc);
        if (lane == 0 && m != kInf) atomicMin(&C->minsucc, (unsigned long long)m);
    }
    if (STATS) {
        const uint64_t s = warp_sum(acc.succ), ins = warp_sum(acc.inserts);
        if (lane == 0 && s) atomicAdd(&C->succ, (unsigned long long)s);
        if (lane == 0 && ins) atomicAdd(&C->inserts, (unsigned long long)ins);
    }
}

// --------------------------------------------------------------------- ExtDist for rho
__device__ uint64_t cta_rho_theta(const RunParams& p, const int32_t* qcur, int32_t q, uint64_t rho, int64_t round,
                                  SelectSmem& sm) {
    if (p.flags & SSSP_RUN_RHO_EXACT) {
        return cta_kth_smallest(QueueKey{qcur, p.dist}, q, rho, sm);
    }
    const uint64_t s = sample_count((uint64_t)q, rho);
    for (uint64_t j = threadIdx.x; j < s; j += blockDim.x) {
        const uint64_t r = splitmix64(p.seed ^ splitmix64(((uint64_t)round << 32) | j));
        p.samples[j] = ld_cg_u64(p.dist + ld_cg_i32(qcur + (int64_t)(r % (uint64_t)q)));
    }
    __syncthreads();
    uint64_t k = (rho * s + (uint64_t)q - 1) / (uint64_t)q;
    k = k < 1 ? 1 : (k > s ? s : k);
    return cta_kth_smallest(ArrayKey{p.samples}, (int64_t)s, k, sm);
}

// --------------------------------------------------------------------- the round loop
template <int POL, bool STATS>
__global__ void __launch_bounds__(kBlock) sssp_round_loop(RunParams p) {
    __shared__ SelectSmem sm;
    Ctrl* ctrl = p.ctrl;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;

    // Alg. 1 lines 1-2: delta[.] = +inf, delta[s] = 0, Q.Update(s)
    for (int64_t i = gtid; i < p.n; i += gsize) p.dist[i] = (i == p.source) ? 0ull : kInf;
    const int64_t nwords = ((int64_t)p.n + 31) >> 5;
    for (int64_t i = gtid; i < nwords; i += gsize)
        p.bm[i] = (i == (p.source >> 5)) ? (1u << (p.source & 31)) : 0u;
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
            const uint64_t minq = a < b ? a : b;  // = min_{v in Q} delta[v], exactly
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
                rho = rho / 10 ? rho / 10 : 1;
            }
            if ((uint64_t)q <= rho) {
                theta = kInf;  // |Q| <= rho: extract all
            } else {
                if (blockIdx.x == 0) {
                    const uint64_t th = cta_rho_theta(p, qcur, q, rho, r, sm);
                    if (threadIdx.x == 0) C->theta = th;
                }
                grid_sync(&ctrl->bar);
                theta = ld_volatile_u64((const uint64_t*)&C->theta);
            }
        }

        // ---- Extract(theta)
        extract_phase<POL, STATS>(p, qcur, qnext, q, theta, C);
        grid_sync(&ctrl->bar);
        // ---- relax N(F) with WriteMin, Update improved vertices
        relax_phase<POL, STATS>(p, qnext, C);
        grid_sync(&ctrl->bar);

        if (STATS && gtid == 0) {
            const unsigned long long hp = C->heavy_pack;
            const int64_t f = (int64_t)C->nlight + (int64_t)(hp >> 32);
            if (p.trace && r - 1 < p.trace_cap) {
                sssp_round* t = p.trace + (r - 1);
                t->qsize = q;
                t->fsize = f;
                t->edges = (int64_t)C->edges;
                t->inserts = (int64_t)C->inserts;
                t->succ = (int64_t)C->succ;
                t->theta = theta;
                t->nheavy = (int64_t)(hp >> 32);
                t->reserved = 0;
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
    int grid[4][2];
};

namespace {

struct Layout {
    uint64_t* dist;
    uint32_t* bm;
    int32_t *q0, *q1;
    FEntry *light, *heavy;
    int32_t *heavy_cb, *chunk_owner;
    uint64_t* samples;
    Ctrl* ctrl;
    int32_t* err;
    size_t bytes;
};

Layout carve(void* base, int32_t n, int64_t m) {
    Carver c(base);
    Layout L;
    const int64_t hcap = std::min<int64_t>(n, m / (kLightMax + 1)) + 1;
    const int64_t ccap = m / kChunk + hcap + 1;
    L.ctrl = c.take<Ctrl>(1);
    L.err = c.take<int32_t>(32);
    L.dist = c.take<uint64_t>(n);
    L.bm = c.take<uint32_t>(((size_t)n + 31) / 32);
    L.q0 = c.take<int32_t>(n);
    L.q1 = c.take<int32_t>(n);
    L.light = c.take<FEntry>(n);
    L.heavy = c.take<FEntry>(hcap);
    L.heavy_cb = c.take<int32_t>(hcap);
    L.chunk_owner = c.take<int32_t>(ccap);
    L.samples = c.take<uint64_t>(kMaxSamples);
    L.bytes = align_up(c.off, 256);
    return L;
}

typedef void (*KernelFn)(RunParams);

KernelFn kernel_for(int pol, bool stats) {
    switch (pol) {
        case SSSP_RHO: return stats ? sssp_round_loop<SSSP_RHO, true> : sssp_round_loop<SSSP_RHO, false>;
        case SSSP_DELTA: return stats ? sssp_round_loop<SSSP_DELTA, true> : sssp_round_loop<SSSP_DELTA, false>;
        case SSSP_BELLMAN_FORD:
            return stats ? sssp_round_loop<SSSP_BELLMAN_FORD, true> : sssp_round_loop<SSSP_BELLMAN_FORD, false>;
        case SSSP_DIJKSTRA:
            return stats ? sssp_round_loop<SSSP_DIJKSTRA, true> : sssp_round_loop<SSSP_DIJKSTRA, false>;
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
    b.bm = L.bm;
    b.q0 = L.q0;
    b.q1 = L.q1;
    b.light = L.light;
    b.heavy = L.heavy;
    b.heavy_cb = L.heavy_cb;
    b.chunk_owner = L.chunk_owner;
    b.samples = L.samples;
    b.ctrl = L.ctrl;
    for (int pol = 0; pol < 4; pol++)
        for (int st = 0; st < 2; st++) {
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kernel_for(pol, st), kBlock, 0);
            if (e != cudaSuccess || per_sm < 1) {
                delete h;
                return e != cudaSuccess ? cuda_error(e, "occupancy query")
                                        : set_error(SSSP_ERR_DEVICE, "round-loop kernel cannot be resident");
            }
            h->grid[pol][st] = per_sm * sms;
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
    KernelFn k = kernel_for(policy, st);
    const int grid = h->grid[policy][st];
    void* args[] = {&p};
    cudaEventRecord(h->ev[0], h->stream);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kBlock), args, 0, h->stream);
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
