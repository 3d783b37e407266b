// loop.cuh — the stepping-algorithm round loop (Alg. 1) as ONE persistent
// cooperative kernel template.  Included by inst.cu (compiled once per policy,
// bidirectional flag and fusion flag, in parallel, possibly with unit-specific constants)
// and by run.cu (host API: layout and launch only).
//
// LaB-PQ of the round loop: the membership flag of a vertex lives in
// the top bit of its delta word (bit 63 set = NOT in Q), the value in the low 63
// bits; the queue is a compacted id array (ping-pong per round).
//   Update(v)   = the WriteMin CAS that lowers the value also clears bit 63; the
//                 thread whose CAS saw bit 63 set appends v (exactly one append per
//                 insertion, no duplicates).
//   Extract(u)  = atomicOr(bit 63): deletes u from Q and returns, atomically, the
//                 value it is relaxed with (its snapshot key).
// Because flag and key share one word, a concurrent WriteMin and Extract can never
// lose an update, so Extract and relax may overlap ("live" rounds, the default).
//
// Append lists (next queue, heavy-chunk descriptors) are SHARDED: kShards segments,
// each with its own counter on its own L2 slice, plus a spill segment.  Same-address
// atomics serialise in the L2 (~7 ns each), so one shared tail counter capped the
// queue scan at ~0.5 TB/s; warps stage appends in shared memory and reserve space in
// their shard once per <= 256 ids.  Readers see a list as the concatenation of its
// segments (prefix of the segment counts, computed per CTA in shared memory).
//
// Per round r:
//   ExtDist  theta_r per policy (Table tab:framework).  rho: every CTA
//            draws the same counter-based samples into shared memory and selects
//            the same theta (readings R5/R6) -> no barrier.
//   Phase A  one pass over the queue (array LaB-PQ P:1011-1012) in tiles
//            (dealt to CTAs, taken by warps from a shared-memory counter; one thin
//            share per warp in fusion kernels): ids with key <= theta are extracted;
//            vertices of degree <= kLight are relaxed by the extracting warp (live) or
//            listed (snapshot mode); heavier ones are cut into kChunk-arc descriptors;
//            the rest of Q is compacted into the next queue.  In live rounds of sparse
//            graphs a WriteMin that reaches a vertex outside Q within theta extracts it
//            on the spot (fusion).                      grid barrier
//   Phase B  warps stride over the chunk descriptors (and, in snapshot mode, the
//            light list): per arc c = d_u + w, filter load of delta[v] (through L1),
//            WriteMin by CAS, append on insertion.  grid barrier (if non-empty)
//   loop while |Q| > 0.
#pragma once
#include <stdio.h>

#include <algorithm>
#include <string.h>

#include "common.cuh"
#include "internal.h"

namespace sssp {

// (a kernel unit is compiled for one fusion flag, INST_FUSE; run.cu sees neither)
#if defined(INST_FUSE) && INST_FUSE
#define SSSP_FUSE_UNIT 1
#else
#define SSSP_FUSE_UNIT 0
#endif
#ifndef SSSP_MIN_BLOCKS
#define SSSP_MIN_BLOCKS 1
#endif
#ifndef SSSP_BLOCK
#define SSSP_BLOCK 1024
#endif
#ifndef SSSP_ARCS
#define SSSP_ARCS 4
#endif
#ifndef SSSP_LIGHT
#define SSSP_LIGHT 32
#endif
constexpr uint64_t kTop = 1ull << 63;        // flag bit: set = not in Q
constexpr uint64_t kVal = kTop - 1;          // value bits of a delta word
constexpr int kBlock = SSSP_BLOCK;           // threads per CTA of the round loop
constexpr int kMinBlocks = SSSP_MIN_BLOCKS;  // CTAs per SM the register budget targets
constexpr int kArcs = SSSP_ARCS;             // arcs per lane in flight
constexpr int kChunk = 32 * kArcs;           // arcs per heavy-chunk descriptor
constexpr int kLight = SSSP_LIGHT;           // out-degree <= kLight: relaxed by the extracting warp
// Shared-memory budget: L1 is what the carveout leaves of the SM's 256 KB, and the carveout
// comes in steps (.., 64, 100, 132, 164, .. KB).  The relax's in-flight loads live in L1 lines,
// so every unit is sized to fall just under a step (DESIGN.md §5 "shared memory per unit"):
// units without fusion 98.8 KB -> the 100 KB step (from 123 KB / 132: rmat24 rho -2.3 %, Delta*
// and BF -3.9 %, rmat20 -2 to -3 %), fusion units 134.9 KB -> 132 (from 164: road graphs -0.5
// to -0.9 %).  What shrank: theta samples held in shared memory (more fall back to CTA 0 and a
// barrier), the per-warp append stage, and the small-round queue.
#ifndef SSSP_SMEM_SAMPLES
#if SSSP_FUSE_UNIT
#define SSSP_SMEM_SAMPLES 480
#else
#define SSSP_SMEM_SAMPLES 512
#endif
#endif
constexpr int kSmemSamples = SSSP_SMEM_SAMPLES;  // theta samples held in shared memory (else CTA-0 fallback)
#ifndef SSSP_RANK_SELECT
#define SSSP_RANK_SELECT 512
#endif
constexpr int kRankSelect = SSSP_RANK_SELECT;  // s <= this: select by rank counting
constexpr int kWarps = kBlock / 32;
#ifndef SSSP_PROF
#define SSSP_PROF 0  // 1: STATS kernels also split phase-A warp time into parts (clock64)
#endif
#ifndef SSSP_SEG_HINT
#define SSSP_SEG_HINT 1  // phase B: find a descriptor's segment by a forward scan from the last one
#endif                   // (0: binary search; the rho unit without fusion uses 0, build.py)
#ifndef SSSP_NEAR_K
#define SSSP_NEAR_K 8
#endif
#ifndef SSSP_FUSE
#define SSSP_FUSE 64
#endif
#ifndef SSSP_ENT
#define SSSP_ENT 2
#endif
constexpr int kEnt = SSSP_ENT;               // queue entries per lane per Extract step (large queues)
#ifndef SSSP_QBUF
#if SSSP_FUSE_UNIT
#define SSSP_QBUF 128
#else
#define SSSP_QBUF 224
#endif
#endif
constexpr int kQBuf = 32 * kArcs > SSSP_QBUF ? 32 * kArcs : SSSP_QBUF;  // staged queue ids per warp (>= 32 * kArcs)
constexpr int kTBuf = 32 * kEnt + 32;        // staged extracted ids per warp
constexpr int kFBuf = 32 * kArcs + 64;       // fused vertices waiting for their relax, per warp
constexpr int kFuseBudget = SSSP_FUSE;       // fused vertices per warp per round (0 = off)
constexpr int kFuseBudgetRho = 96;           // the same for rho-stepping (bounded depth, run.cu)
// Default bound on the hops a local search may go from its extracted seed (DESIGN.md §5
// "fusion depth"; the paper bounds its local search by t = 4096 visited vertices).  A
// round lasts as long as its slowest warp's local search: for rho-stepping, whose theta follows
// the queue, 10 hops (with the per-warp budget of 64) cut grid4096 by 23 %, rgg4m by 14 % and
// grid256 by 23 %.  Delta*-stepping's theta advances by Delta whatever the searches reached, so
// a bound there can leave them behind theta (grid4096 Delta* 2^17 at 8 hops: 932 -> 2,706 rounds
// of Bellman-Ford-like re-relaxation); its default stays unbounded (run.cu).
#ifndef SSSP_FUSE_DEPTH_RHO
#define SSSP_FUSE_DEPTH_RHO 10
#endif
constexpr int kFuseDepthRho = SSSP_FUSE_DEPTH_RHO;
constexpr int kFuseDepth = 1 << 30;  // unbounded
constexpr int kFuseMaxDeg = 1024;            // a fused vertex of higher degree goes back to Q
constexpr int kContigTiles = 16;             // queue < kContigTiles*32 ids per warp: contiguous shares
constexpr int kSparseDeg = 20;               // fusion in rounds whose frontier averages < 20 arcs
constexpr int kShards = 32;                  // append-list segments (+1 spill)
constexpr int kSeg = kShards + 1;
constexpr int kCntStride = 256;              // int32 words between counters (1 KB: distinct L2 slices)
constexpr int kMaxCtas = 4096;
constexpr int kPolicies = 5;
constexpr int kProf = 8;                     // SSSP_PROF counters per round
constexpr int kNearK = SSSP_NEAR_K;          // near queue target: ~kNearK rounds of extraction
#ifndef SSSP_FAR_SAMPLES
#define SSSP_FAR_SAMPLES 256
#endif
constexpr int kFarSamples = SSSP_FAR_SAMPLES; // vertices probed to place a new near/far split (<= kRankSelect
                                              // far keys: a rank-count select, no radix passes)
static_assert(32 * kArcs <= kQBuf, "one relax step must fit the stage");
static_assert(kBlock % 32 == 0 && kBlock <= 1024, "block size");

// A vertex (or a piece of one) to relax: snapshot key and a CSR arc range.
struct __align__(16) Desc {
    uint64_t d;
    int32_t beg;
    int32_t len;
};

// Per-round control (triple-buffered by round slot).
struct __align__(128) RoundCnt {
    int32_t nlight;              // snapshot mode: light frontier entries
    int32_t nheavy;              // STATS: heavy vertices
    unsigned long long theta;    // CTA-0 fallback theta
    unsigned long long fsize;    // STATS: extracted
    unsigned long long edges;    // STATS: arcs of extracted vertices
    unsigned long long succ;     // STATS: successful WriteMins
    unsigned long long inserts;  // STATS: ids inserted into Q by relax
    unsigned long long split;    // CTA-0 broadcast of a new near/far split
    unsigned long long busy_a;   // STATS: sum over warps of phase-A busy time (ns)
    unsigned long long busy_b;   // STATS: same for phase B
    unsigned long long busy_a_max;  // STATS: slowest warp's phase-A busy time (ns)
    unsigned long long fused;    // STATS: vertices extracted by fusion
    unsigned long long prof[kProf];  // SSSP_PROF: phase-A warp sums (see Warp::prof)
};

struct __align__(128) Ctrl {
    RoundCnt cnt[3];
    // results (copied to the host after the run)
    int32_t status;
    int32_t pad1;
    int64_t rounds;
    int64_t tot_extracted, tot_edges, tot_succ, tot_inserts, tot_qscan, max_q, max_f, tot_dense;
    // small-frontier rounds: the state CTA 0 hands back to the grid
    int32_t sm_epoch;         // incremented (release) at every hand-back
    int32_t sm_end;           // 1: the run is over (Q empty or max_rounds exceeded)
    int64_t sm_r;             // round the grid resumes at
    int64_t sm_qtot;          // |Q| at that round (all of it listed in the queue array)
    uint64_t sm_theta_prev;   // Delta* / Delta-stepping: last theta
    int32_t sm_warm;          // rho: warm-up rounds used
    int32_t sm_rounds;        // STATS: rounds run by CTA 0
};

// A sharded append list: segment s < kShards holds [s*cap, s*cap + min(count_s, cap)),
// the spill segment [kShards*cap, ...).  Counters live 1 KB apart.
template <typename T>
struct Sharded {
    T* base;
    int32_t* cnt;       // cnt[s * kCntStride]
    int64_t cap;        // per-shard capacity
    int64_t spill_cap;  // capacity of the spill segment
    int32_t* err;       // set to SSSP_ERR_INTERNAL if a reservation ever exceeded the spill
    __device__ __forceinline__ T* seg(int s) const { return base + (int64_t)s * cap; }
    __device__ __forceinline__ int64_t seg_count(int s) const {
        const int64_t c = __ldcg(cnt + s * kCntStride);
        return s < kShards ? (c < cap ? c : cap) : c;
    }
};

struct RunParams {
    int32_t n;
    int32_t source;
    int64_t m;
    const int32_t* __restrict__ off;
    const uint2* __restrict__ arc;  // interleaved CSR arcs {head, weight} (workspace copy)
    // isolated-vertex compaction (run.cu build_compaction): the run works on ids 0..n-1
    // (the non-isolated vertices); nofo / ofno map caller ids <-> run ids, `out` is the
    // caller's distance array of n_out entries.  nofo == nullptr: no compaction, dist is
    // the caller's array
    const int32_t* nofo;
    const int32_t* ofno;
    uint64_t* out;
    int32_t n_out;
    uint64_t* dist;
    int32_t* qbuf[2];   // queue storage, ping-pong
    int64_t qcap;       // per-shard queue capacity
    Desc* chunks;       // chunk descriptor storage
    int64_t ccap;       // per-shard chunk capacity
    int64_t cspill;     // chunk spill capacity
    int32_t* counters;  // [3 slots][2 lists: queue, chunks][kSeg] * kCntStride
    uint64_t* cta_min;  // [3 slots][kMaxCtas]: per-CTA min for Delta / Dijkstra
    int64_t* cta_delta; // [3 slots][kMaxCtas]: per-CTA change of |Q| (inserts - extractions)
    int32_t* cta_ext;   // [3 slots][kMaxCtas]: per-CTA extractions (fusion included)
    Desc* light;
    uint64_t* samples;
    Ctrl* ctrl;
    uint64_t param;
    uint32_t flags;
    uint64_t seed;
    int64_t max_rounds;
    sssp_round* trace;
    int64_t trace_cap;
    int32_t* ext_count;
    int32_t fuse_budget;  // fused vertices per warp per round (FUSE kernels)
    int32_t fuse_depth;   // hops from the extracted seed a fused vertex may lie (FUSE kernels)
};

__device__ __forceinline__ int32_t* counters_of(const RunParams& p, int slot, int list) {
    return p.counters + (int64_t)((slot * 2 + list) * kSeg) * kCntStride;
}
__device__ __forceinline__ Sharded<int32_t> queue_of(const RunParams& p, int64_t round_of_queue) {
    // Q_r lives in qbuf[r & 1]; its counts are in slot (r + 2) % 3
    return Sharded<int32_t>{p.qbuf[round_of_queue & 1], counters_of(p, (int)((round_of_queue + 2) % 3), 0), p.qcap,
                            (int64_t)p.n, &p.ctrl->status};
}
__device__ __forceinline__ Sharded<Desc> chunks_of(const RunParams& p, int64_t r) {
    return Sharded<Desc>{p.chunks, counters_of(p, (int)(r % 3), 1), p.ccap, p.cspill, &p.ctrl->status};
}

__device__ __forceinline__ void reset_cnt(RoundCnt* c) {
    c->nlight = 0;
    c->nheavy = 0;
    c->theta = 0;
    c->fsize = 0;
    c->edges = 0;
    c->succ = 0;
    c->inserts = 0;
    c->split = 0;
    c->busy_a = 0;
    c->busy_b = 0;
    c->busy_a_max = 0;
    c->fused = 0;
    for (int i = 0; i < kProf; i++) c->prof[i] = 0;
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

// Filter read of delta[v] for a relaxation: through L1 (hub targets are shared by many
// arcs of an SM).  A stale L1 copy can only be higher than the current value (delta only
// decreases, and every grid barrier's fence invalidates L1), so it can only cause a CAS
// that then fails and retries with the word the CAS returned: never a lost update.
__device__ __forceinline__ uint64_t dist_filter_ld(const uint64_t* p) {
    // (.cg, L1::no_allocate and L1::evict_first measured after the L1 resize: rmat24 rho +0.2 % /
    // +18 % / +18 %, BF +3 % / +28 % / +25 %, rmat20 +4 to +38 %)
    return __ldca((const unsigned long long*)p);
}

__host__ __device__ constexpr bool uses_min(int pol) {
    return pol == SSSP_DELTA || pol == SSSP_DIJKSTRA || pol == SSSP_DELTA_STEPPING;
}

// --------------------------------------------------------------------- segment prefix
// Exclusive prefix of a sharded list's segment counts, in shared memory (pref[kSeg] =
// total).  Called by all threads; ends with __syncthreads.
template <typename T>
__device__ __forceinline__ void load_prefix(const Sharded<T>& L, int64_t* pref) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t c0 = L.seg_count(lane);                     // shards 0..31
        const int64_t c1 = lane == 0 ? L.seg_count(kShards) : 0;  // spill
        int64_t x = c0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += t;
        }
        const int64_t spill = __shfl_sync(kFull, c1, 0);
        pref[lane] = x - c0;
        if (lane == 31) {
            pref[kShards] = x;
            pref[kSeg] = x + spill;
        }
    }
    __syncthreads();
}
static_assert(kShards == 32, "load_prefix assumes one warp of shards");

// segment of virtual index i < total: largest s with pref[s] <= i (pref is smem)
__device__ __forceinline__ int seg_of(const int64_t* pref, int64_t i) {
    int s = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)
        if (s + step <= kShards && pref[s + step] <= i) s += step;
    return s;
}

// --------------------------------------------------------------------- per-warp staging
constexpr int kPend = 64;  // deferred WriteMins: pending WriteMins per warp (drained at 32)
struct WarpStage {
    Desc nd[2];           // phase B (dynamic items): the next chunk descriptor, copied in by cp.async
#if !SSSP_FUSE_UNIT
    int32_t ext;          // vertices this warp extracted this round (lane 0 counts; small-round entry test)
    int32_t snxt;         // small rounds: which s_small.q[] this warp appends Q_{r+1} to
#endif
    int32_t take[kTBuf];  // ids that pass the theta test, extracted 32 at a time
    int32_t q[kQBuf];     // ids appended to the next queue
#if !defined(INST_BIDIR) || INST_BIDIR
    uint64_t mins[32];    // bidirectional relaxation: per-vertex pulled minimum
#endif
#if !SSSP_FUSE_UNIT
    uint64_t pc[kPend];   // deferred WriteMins (kernels without fusion or pull): candidate ...
    uint64_t pw[kPend];   // ... the word the filter read ...
    int32_t pv[kPend];    // ... and the target
#endif
};
// (a unit's shared memory holds only the stage fields its kernels use: the rest of the 256 KB
// of L1 / shared memory caches the filter reads of delta)
struct FuseStage {        // FUSE kernels only (kept out of the others' shared memory, which is L1)
    uint64_t fd[kFBuf];   // fused vertices: key ...
    int32_t fid[kFBuf];   // ... id ...
    int32_t fdep[kFBuf];  // ... and hops from the extracted seed
};

// --------------------------------------------------------------------- small-frontier rounds
// While |Q| <= kSmallQ (all of it listed) and a round's frontier has at most kSmallArcs arcs,
// CTA 0 runs the rounds alone with CTA barriers and the queue in shared memory; the other
// CTAs wait on a flag (DESIGN.md §5 "small-frontier rounds"; the paper's "insufficient
// workload and thus overhead in the synchronization cost").
#ifndef SSSP_SMALL
#define SSSP_SMALL 1  // 0: compile the small-frontier path out (A/B builds)
#endif
// Kernels with fusion do not run small rounds: there a small |Q| hides the fused work, and the
// path cost them 3-6 % (A/B on grid256 / grid4096 / rgg4m); the others gain from it.
__host__ __device__ constexpr bool small_on(bool fuse) { return SSSP_SMALL && !fuse; }
#ifndef SSSP_SMALL_Q
#define SSSP_SMALL_Q 1024
#endif
constexpr int kSmallQ = SSSP_SMALL_Q;
constexpr int kSmallArcs = 32768;
#ifndef SSSP_SMALL_F
#define SSSP_SMALL_F 256
#endif
constexpr int kSmallF = SSSP_SMALL_F;  // ... entered only after a round that extracted at most this many
                               // vertices (fusion included), left after one that extracted more
                               // than 2 kSmallF: on road graphs a small |Q| can still fuse tens of
                               // thousands of vertices per round, more than one SM should take
static_assert(kSmallQ % kBlock == 0, "small-round queue: whole entries per thread");
struct SmallSmem {
    int32_t q[2][kSmallQ];     // Q_r / Q_{r+1} ids (entries >= kSmallQ of Q_{r+1} go to gq)
    int32_t qcnt[2];
    int32_t on;                // 1 while CTA 0 runs small rounds: wq_flush appends here
    int32_t* gq[2];            // q[k]'s continuation in the grid's flat layout (overflow, hand-back)
    int64_t qcap;
    // per-round scalars, by round parity (a round resets its own before its first barrier
    // while the previous round's may still be read: no barrier between rounds)
    unsigned long long arcs[2];  // arcs of the round's frontier
    int32_t heavy[2];            // a vertex of degree > kLight was extracted (chunk list in use)
    int32_t ext[2];              // vertices extracted this round (fusion included)
};
#if !SSSP_FUSE_UNIT
__shared__ SmallSmem s_small;
#endif

// i-th entry of a queue buffer seen as one flat list: shard-0 segment, then the spill segment
__device__ __forceinline__ int32_t* flat_slot(int32_t* base, int64_t qcap, int64_t i) {
    return i < qcap ? base + i : base + (int64_t)kShards * qcap + (i - qcap);
}

// dynamic shared memory: per-warp stages, theta samples, select scratch [, fuse stages]
constexpr size_t kSmemBase = (kWarps * sizeof(WarpStage) + kSmemSamples * sizeof(uint64_t) + sizeof(SelectSmem) + 15) /
                             16 * 16;
extern __shared__ __align__(16) unsigned char sssp_dyn_smem[];

struct Acc {
    uint64_t minsucc = kInf;
    uint32_t succ = 0;
    uint32_t inserts = 0;
    uint32_t fused = 0;        // STATS: vertices extracted by fusion
    uint64_t fused_edges = 0;  // STATS: their arcs
};

// Per-round values every warp of a CTA reads.  Kernels without fusion keep them in shared
// memory (written by thread 0 before a CTA barrier), not in each thread's registers: they run
// at 64 registers, and this cold state cost them spills in their hot loops (Bellman-Ford on
// rmat24 +16 % with the small-round path).  The fusion kernels, whose hops are latency chains,
// keep the round-1 layout: per-thread registers (A/B: 3-12 % slower from shared memory).
struct RoundSmem {
    Sharded<int32_t> qnext;  // the list WriteMins append Q_{r+1}'s near part to
    RoundCnt* C;             // this round's counters (STATS, snapshot light list)
};
__shared__ RoundSmem s_rnd;

struct Warp {  // per-warp working state in registers (qn, fn, pn are warp-uniform)
#if SSSP_FUSE_UNIT
    WarpStage* st_;
    FuseStage* fs_;
    Sharded<int32_t> qnext_;
    RoundCnt* C_;
    int shard_;
    __device__ __forceinline__ WarpStage* st() const { return st_; }
    __device__ __forceinline__ FuseStage* fs() const { return fs_; }
    __device__ __forceinline__ const Sharded<int32_t>& qnext() const { return qnext_; }
    __device__ __forceinline__ RoundCnt* C() const { return C_; }
    __device__ __forceinline__ int shard() const { return shard_; }
    __device__ __forceinline__ void init() {
        st_ = (WarpStage*)sssp_dyn_smem + (threadIdx.x >> 5);
        fs_ = (FuseStage*)(sssp_dyn_smem + kSmemBase) + (threadIdx.x >> 5);
        shard_ = (int)(warp_rank() % kShards);
    }
    // every thread, at the round top
    __device__ __forceinline__ void set_round(const Sharded<int32_t>& q, RoundCnt* c) {
        qnext_ = q;
        C_ = c;
    }
    __device__ __forceinline__ Sharded<int32_t> swap_qnext(const Sharded<int32_t>& q) {  // all threads
        const Sharded<int32_t> o = qnext_;
        qnext_ = q;
        return o;
    }
#else
    __device__ __forceinline__ WarpStage* st() const { return (WarpStage*)sssp_dyn_smem + (threadIdx.x >> 5); }
    __device__ __forceinline__ FuseStage* fs() const {
        return (FuseStage*)(sssp_dyn_smem + kSmemBase) + (threadIdx.x >> 5);
    }
    __device__ __forceinline__ const Sharded<int32_t>& qnext() const { return s_rnd.qnext; }
    __device__ __forceinline__ RoundCnt* C() const { return s_rnd.C; }
    __device__ __forceinline__ int shard() const { return (int)(warp_rank() % kShards); }
    __device__ __forceinline__ void init() {}
    // every thread, at the round top, before a CTA barrier
    __device__ __forceinline__ void set_round(const Sharded<int32_t>& q, RoundCnt* c) {
        if (threadIdx.x == 0) {
            s_rnd.qnext = q;
            s_rnd.C = c;
        }
    }
    __device__ __forceinline__ Sharded<int32_t> swap_qnext(const Sharded<int32_t>& q) {  // all threads
        Sharded<int32_t> o = s_rnd.qnext;
        __syncthreads();
        if (threadIdx.x == 0) s_rnd.qnext = q;
        __syncthreads();
        return o;
    }
#endif
    uint64_t split;       // near/far split: keys <= split are held in the queue array
    uint64_t fuse_theta;  // live rounds: theta (a vertex outside Q improved to <= theta is
                          // extracted on the spot, DESIGN.md §5 "fusion"); 0 = no fusion
    int64_t qdelta;       // this lane's inserts - extractions (|Q| bookkeeping)
    int32_t qn;
    int32_t fn;       // staged fused vertices (warp-uniform)
    int32_t fbudget;  // fusions left this round (warp-uniform)
    int32_t pn;       // deferred WriteMins: pending (warp-uniform)
    Acc acc;
#if SSSP_PROF
    // cycles in scan, take, light relax, queue flush, fuse_drain; fuse_drain batches;
    // relax steps (relax_slots calls); cycles in relax_slots
    uint64_t prof[kProf];
#endif
};

// SSSP_PROF: add the cycles since t0 to part i of the warp's phase-A profile
#if SSSP_PROF
#define PROF_T0(t) const long long t = clock64()
#define PROF_ADD(W, i, t) ((W).prof[i] += (uint64_t)(clock64() - (t)))
#else
#define PROF_T0(t)
#define PROF_ADD(W, i, t)
#endif

// A successful WriteMin replaced word w_old by value c (flag cleared).  Returns true iff
// v must be appended to the near queue: it was outside Q (insertion) and c <= split, or
// it was a far member of Q (value > split) that now falls into the near range.
template <bool STATS>
__device__ __forceinline__ bool admit(uint64_t w_old, uint64_t c, Warp& W) {
    if (w_old & kTop) {
        W.qdelta++;
        if (STATS) W.acc.inserts++;
        return c <= W.split;
    }
    return (w_old & kVal) > W.split && c <= W.split;
}

// Reserve `tot` slots of a sharded list for this warp (lane 0 does the atomics).
// Element i < tot goes to p0 + i if i < fit, else to p1 + (i - fit) (spill segment).
// The capacities make overflow impossible (a list never holds more than its bound), but a
// reservation past the spill segment is still refused: `lim` < tot elements are writable
// and the run fails with SSSP_ERR_INTERNAL instead of corrupting memory.
template <typename T>
__device__ __forceinline__ void reserve(const Sharded<T>& L, int shard, int32_t tot, T*& p0, int32_t& fit, T*& p1,
                                        int32_t& lim) {
    int64_t pos = 0, spos = 0;
    if (lane_id() == 0) {
        pos = atomicAdd(L.cnt + shard * kCntStride, tot);
        const int64_t f = pos >= L.cap ? 0 : (L.cap - pos < tot ? L.cap - pos : tot);
        if (f < tot) spos = atomicAdd(L.cnt + kShards * kCntStride, (int32_t)(tot - f));
    }
    pos = __shfl_sync(kFull, pos, 0);
    spos = __shfl_sync(kFull, spos, 0);
    fit = pos >= L.cap ? 0 : (int32_t)(L.cap - pos < tot ? L.cap - pos : tot);
    const int64_t room = L.spill_cap - spos;
    lim = fit + (int32_t)(room <= 0 ? 0 : (room < tot - fit ? room : tot - fit));
    if (lim < tot && lane_id() == 0) atomicExch(L.err, (int32_t)SSSP_ERR_INTERNAL);
    p0 = L.seg(shard) + pos;
    p1 = L.seg(kShards) + spos;
}

__device__ __forceinline__ void wq_flush(Warp& W) {
    if (W.qn == 0) return;
    PROF_T0(tf);
    __syncwarp();
#if !SSSP_FUSE_UNIT
    if (s_small.on) {  // small-frontier rounds (CTA 0 alone): Q_{r+1} in shared memory
        int32_t pos = 0;
        const int nx = W.st()->snxt;
        if (lane_id() == 0) pos = atomicAdd(&s_small.qcnt[nx], W.qn);
        pos = __shfl_sync(kFull, pos, 0);
        int32_t* sq = s_small.q[nx];
        for (int32_t i = lane_id(); i < W.qn; i += 32) {
            const int32_t v = W.st()->q[i], j = pos + i;
            if (j < kSmallQ)
                sq[j] = v;
            else
                *flat_slot(s_small.gq[nx], s_small.qcap, j) = v;
        }
        __syncwarp();
        W.qn = 0;
        return;
    }
#endif
    int32_t *p0, *p1;
    int32_t fit, lim;
    reserve(W.qnext(), W.shard(), W.qn, p0, fit, p1, lim);
    for (int32_t i = lane_id(); i < lim; i += 32) {
        const int32_t v = W.st()->q[i];
        if (i < fit)
            p0[i] = v;
        else
            p1[i - fit] = v;
    }
    __syncwarp();
    W.qn = 0;
    PROF_ADD(W, 3, tf);
}

// stage the lanes' ids with pred (one id per lane)
__device__ __forceinline__ void wq_push1(Warp& W, bool pred, int32_t id) {
    const uint32_t mask = __ballot_sync(kFull, pred);
    if (!mask) return;
    const int32_t cnt = __popc(mask);
    if (W.qn + cnt > kQBuf) wq_flush(W);
    if (pred) W.st()->q[W.qn + __popc(mask & lanemask_lt())] = id;
    W.qn += cnt;
}

// --------------------------------------------------------------------- relax
// Outcome of a relaxation slot.
enum { kNone = 0, kAppend = 1, kFused = 2 };

// The word a successful WriteMin of c over word w writes: c with the flag cleared (v is
// in Q), or - when fusing - c with the flag still set (v was outside Q and is extracted
// on the spot by this warp, so it never enters Q).
__device__ __forceinline__ bool fuses(bool fuse, uint64_t w, uint64_t c, const Warp& W) {
    return fuse && (w & kTop) && c <= W.fuse_theta;
}
// FUSE kernels: slot t of a relax step may fuse (its source vertex lies < fuse_depth hops from
// its extracted seed) iff bit t of the step's mask is set

// WriteMin(delta[v], c) on the packed word, given a prior read `w`: CAS retries.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ int write_min(uint64_t* dist, int32_t v, uint64_t c, uint64_t w, bool fuse, Warp& W) {
    while ((w & kVal) > c) {
        const bool f = fuses(fuse, w, c, W);
        const uint64_t old = atomicCAS((unsigned long long*)(dist + v), (unsigned long long)w,
                                       (unsigned long long)(f ? (c | kTop) : c));
        if (old == w) {
            if (STATS) W.acc.succ++;
            if (f) return kFused;
            if (uses_min(POL)) W.acc.minsucc = c < W.acc.minsucc ? c : W.acc.minsucc;
            return admit<STATS>(w, c, W) ? kAppend : kNone;
        }
        w = old;
    }
    return kNone;
}

// Deferred WriteMins: run the `cnt` newest pending ones, one per lane (one CAS round trip
// for up to 32 of them), and stage the inserted ids.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void run_pending(const RunParams& p, Warp& W, int32_t cnt) {
#if !SSSP_FUSE_UNIT
    const int lane = lane_id();
    __syncwarp();
    int out = kNone;
    int32_t v = -1;
    if (lane < cnt) {
        const int32_t j = W.pn - cnt + lane;
        v = W.st()->pv[j];
        out = write_min<POL, STATS, FUSE, BIDIR>(p.dist, v, W.st()->pc[j], W.st()->pw[j], false, W);
    }
    __syncwarp();
    W.pn -= cnt;
    wq_push1(W, out == kAppend, v);
#endif
}
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void drain_pending(const RunParams& p, Warp& W) {
    while (!FUSE && !BIDIR && W.pn > 0) run_pending<POL, STATS, FUSE, BIDIR>(p, W, W.pn < 32 ? W.pn : 32);
}

// Relax kArcs arcs per lane (v < 0 = empty slot): filter loads, WriteMins, stage the
// inserted ids (Alg. 1 lines 5-6).
struct NoPull {
    __device__ __forceinline__ void operator()(const int32_t (&)[kArcs], const uint64_t (&)[kArcs], uint64_t (&)[kArcs]) {}
};

template <int POL, bool STATS, bool FUSE, bool BIDIR, typename Pull = NoPull>
__device__ __forceinline__ void relax_slots(const RunParams& p, const int32_t (&v)[kArcs], uint64_t (&c)[kArcs],
                                            Warp& W, uint32_t fok = ~0u, const int32_t* cdep = nullptr,
                                            Pull pull = Pull()) {
    PROF_T0(trs);
#if SSSP_PROF
    W.prof[6]++;
#endif
    // room for a full step of fusions and budget left (warp-uniform)
    const bool fuse = FUSE && W.fuse_theta != 0 && W.fbudget > 0 && W.fn <= kFBuf - 32 * kArcs;
    uint64_t cur[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) cur[t] = v[t] >= 0 ? dist_filter_ld(p.dist + v[t]) : 0ull;
    pull(v, cur, c);  // bidirectional relaxation may lower the candidates (SURVEY f-2)
#if !SSSP_FUSE_UNIT
    if constexpr (!FUSE && !BIDIR) {
        // Deferred WriteMins: the improving candidates (a few per step in bulk rounds) are
        // staged and their CAS issued 32 at a time, so a step waits on its key gathers only,
        // not also on a CAS round trip.  Any order of WriteMins is valid, and the CAS
        // re-checks the word it expects (a change in between just retries).
#pragma unroll
        for (int t = 0; t < kArcs; t++) {
            const bool imp = v[t] >= 0 && (cur[t] & kVal) > c[t];
            const uint32_t m = __ballot_sync(kFull, imp);
            if (!m) continue;
            if (imp) {
                const int32_t j = W.pn + __popc(m & lanemask_lt());
                W.st()->pv[j] = v[t];
                W.st()->pc[j] = c[t];
                W.st()->pw[j] = cur[t];
            }
            W.pn += __popc(m);
            if (W.pn >= 32) run_pending<POL, STATS, FUSE, BIDIR>(p, W, 32);
        }
        PROF_ADD(W, 7, trs);
        return;
    } else
#endif
    {
    // first CAS attempt of every slot issued back to back (one round trip, not kArcs),
    // then the rare retries
    uint64_t old[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++)
        old[t] = (v[t] >= 0 && (cur[t] & kVal) > c[t])
                     ? atomicCAS((unsigned long long*)(p.dist + v[t]), (unsigned long long)cur[t],
                                 (unsigned long long)(fuses(fuse && ((fok >> t) & 1), cur[t], c[t], W) ? (c[t] | kTop) : c[t]))
                     : cur[t] + 1;  // "no attempt" marker: != cur[t]
    int32_t cnt = 0, fcnt = 0;
    int out[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) {
        out[t] = kNone;
        if (v[t] >= 0 && (cur[t] & kVal) > c[t]) {
            if (old[t] == cur[t]) {
                if (STATS) W.acc.succ++;
                if (fuses(fuse && ((fok >> t) & 1), cur[t], c[t], W)) {
                    out[t] = kFused;
                } else {
                    if (uses_min(POL)) W.acc.minsucc = c[t] < W.acc.minsucc ? c[t] : W.acc.minsucc;
                    out[t] = admit<STATS>(cur[t], c[t], W) ? kAppend : kNone;
                }
            } else {
                out[t] = write_min<POL, STATS, FUSE, BIDIR>(p.dist, v[t], c[t], old[t], fuse && ((fok >> t) & 1), W);
            }
        }
        cnt += out[t] == kAppend;
        fcnt += out[t] == kFused;
    }
    constexpr int kCntBits = kArcs < 8 ? 3 : (kArcs < 16 ? 4 : 5);  // per-lane count bits
    static_assert(kArcs < 32, "per-lane counts");
    if (__any_sync(kFull, cnt != 0)) {
        int32_t tot;
        const int32_t excl = warp_excl_scan_small<kCntBits>(cnt, tot);
        if (W.qn + tot > kQBuf) wq_flush(W);
        int32_t pos = W.qn + excl;
#pragma unroll
        for (int t = 0; t < kArcs; t++)
            if (out[t] == kAppend) W.st()->q[pos++] = v[t];
        W.qn += tot;
    }
    if (FUSE && fuse && __any_sync(kFull, fcnt != 0)) {
        int32_t tot;
        const int32_t excl = warp_excl_scan_small<kCntBits>(fcnt, tot);
        int32_t pos = W.fn + excl;
#pragma unroll
        for (int t = 0; t < kArcs; t++)
            if (out[t] == kFused) {
                W.fs()->fid[pos] = v[t];
                W.fs()->fd[pos] = c[t];
                W.fs()->fdep[pos] = cdep[t];
                pos++;
            }
        W.fn += tot;
        W.fbudget -= tot;
    }
    PROF_ADD(W, 7, trs);
    }
}

// One chunk: arcs [beg, beg+len) of a vertex with key d, len <= kChunk.  Lane-strided
// so every load instruction of the warp reads 128 contiguous bytes.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void relax_chunk(const RunParams& p, uint64_t d, int32_t beg, int32_t len, Warp& W) {
    const int lane = lane_id();
    int32_t v[kArcs];
    uint64_t c[kArcs];
#pragma unroll
    for (int t = 0; t < kArcs; t++) {
        const int32_t k = t * 32 + lane;
        const uint2 a = k < len ? ld_stream_arc(p.arc + beg + k) : make_uint2(0xFFFFFFFFu, 0u);
        v[t] = (int32_t)a.x;
        c[t] = d + a.y;
    }
    int32_t cd[kArcs];  // a chunk's vertex was extracted from Q: its targets lie 1 hop from it
#pragma unroll
    for (int t = 0; t < kArcs; t++) cd[t] = 1;
    relax_slots<POL, STATS, FUSE, BIDIR>(p, v, c, W, ~0u, cd);
}

// Up to 32 vertices, one per lane (deg = 0 for none): the warp walks their
// concatenated arc lists; arc e belongs to the largest lane o with excl[o] <= e.
// Bidirectional relaxation (paper P:1360-1366, SURVEY f-2; undirected graphs only): the
// keys gathered for the filter are the neighbours' tentative distances, so before
// pushing, each vertex u of the step first pulls delta[u] <- min_v delta[v] + w(v,u) over
// the step's arcs, lowers delta[u] (keeping its flag bit) and pushes with the lower key.
struct BidirPull {
    const RunParams* p;
    uint64_t* mins;  // per-warp shared memory [32]
    const int32_t* o;
    const uint32_t* wt;
    uint64_t* d;  // this lane's vertex key (updated)
    int32_t uid;  // this lane's vertex id, -1 if none
    __device__ __forceinline__ void operator()(const int32_t (&v)[kArcs], const uint64_t (&cur)[kArcs],
                                               uint64_t (&c)[kArcs]) {
        const int lane = lane_id();
        mins[lane] = kInf;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kArcs; t++)
            if (v[t] >= 0 && (cur[t] & kVal) != kVal)
                atomicMin((unsigned long long*)(mins + o[t]), (unsigned long long)((cur[t] & kVal) + wt[t]));
        __syncwarp();
        const uint64_t best = mins[lane];
        if (uid >= 0 && best < *d) {
            uint64_t w = __ldcg((const unsigned long long*)(p->dist + uid));
            while ((w & kVal) > best) {
                const uint64_t old = atomicCAS((unsigned long long*)(p->dist + uid), (unsigned long long)w,
                                               (unsigned long long)((w & kTop) | best));
                if (old == w) {
                    w = (w & kTop) | best;
                    break;
                }
                w = old;
            }
            *d = (w & kVal) < best ? (w & kVal) : best;
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kArcs; t++) {
            const uint64_t od = __shfl_sync(kFull, *d, o[t]);
            if (v[t] >= 0) c[t] = od + wt[t];
        }
    }
};

// FUSE kernels: `dep` = hops of this lane's vertex from its extracted seed (0 for a vertex
// extracted from Q); a vertex it reaches may be fused only while dep + 1 <= fuse_depth.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void relax_vertices(const RunParams& p, uint64_t d, int32_t beg, int32_t deg, Warp& W,
                                               int32_t uid = -1, int32_t dep = 0) {
    const int lane = lane_id();
    if (__all_sync(kFull, deg <= kArcs)) {
        // every vertex fits one lane: lane-local arcs, no scan or owner search (fusion
        // chains on grids are latency chains: A/B grid4096 Delta* 63.2 -> 59.0 ms, grid256
        // -4 %, rgg4m +1.5-2.7 %, rmat20/24 within 1 %)
        int32_t v[kArcs], o[kArcs];
        uint32_t wt[kArcs];
        uint64_t c[kArcs];
#pragma unroll
        for (int t = 0; t < kArcs; t++) {
            const uint2 a = t < deg ? ld_stream_arc(p.arc + beg + t) : make_uint2(0xFFFFFFFFu, 0u);
            v[t] = (int32_t)a.x;
            wt[t] = a.y;
            c[t] = d + a.y;
            o[t] = lane;
        }
        int32_t cd[kArcs];
#pragma unroll
        for (int t = 0; t < kArcs; t++) cd[t] = dep + 1;
        const uint32_t fok = (FUSE && dep + 1 > p.fuse_depth) ? 0u : ~0u;
#if !defined(INST_BIDIR) || INST_BIDIR
        if (BIDIR && __any_sync(kFull, uid >= 0))
            relax_slots<POL, STATS, FUSE, BIDIR>(p, v, c, W, fok, cd, BidirPull{&p, W.st()->mins, o, wt, &d, uid});
        else
#endif
            relax_slots<POL, STATS, FUSE, BIDIR>(p, v, c, W, fok, cd);
        return;
    }
    int32_t total, excl;
    if (__all_sync(kFull, deg < 64)) {  // light vertices (degree <= 32): bit-plane scan
        excl = warp_excl_scan_small<6>(deg, total);
    } else {
        const int32_t incl = warp_incl_scan(deg);
        total = __shfl_sync(kFull, incl, 31);
        excl = incl - deg;
    }
    const int32_t rowbase = beg - excl;  // CSR position of concatenated arc e of this lane = rowbase + e
    const bool bidir = BIDIR && __any_sync(kFull, uid >= 0);
    for (int32_t s0 = 0; s0 < total; s0 += 32 * kArcs) {
        int32_t v[kArcs], o[kArcs];
        uint32_t wt[kArcs];
        uint64_t c[kArcs];
        // pull only into a vertex whose whole arc list is in this step: arcs pushed in an
        // earlier step with a higher key would otherwise never see the lower one
        const int32_t uid_step = (excl >= s0 && excl + deg <= s0 + 32 * kArcs) ? uid : -1;
#pragma unroll
        for (int t = 0; t < kArcs; t++) {
            const int32_t e = s0 + t * 32 + lane;
            o[t] = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int32_t x = __shfl_sync(kFull, excl, o[t] + step);
                if (x <= e) o[t] += step;
            }
            const int32_t rb = __shfl_sync(kFull, rowbase, o[t]);
            const uint64_t od = __shfl_sync(kFull, d, o[t]);
            const bool ok = e < total;
            const uint2 a = ok ? ld_stream_arc(p.arc + rb + e) : make_uint2(0xFFFFFFFFu, 0u);
            v[t] = (int32_t)a.x;
            wt[t] = a.y;
            c[t] = od + wt[t];
        }
        int32_t cd[kArcs];
        uint32_t fok = 0;
        if (FUSE) {
#pragma unroll
            for (int t = 0; t < kArcs; t++) {
                cd[t] = __shfl_sync(kFull, dep, o[t]) + 1;
                fok |= (cd[t] <= p.fuse_depth ? 1u : 0u) << t;
            }
        }
#if !defined(INST_BIDIR) || INST_BIDIR
        if (BIDIR && bidir)
            relax_slots<POL, STATS, FUSE, BIDIR>(p, v, c, W, fok, cd, BidirPull{&p, W.st()->mins, o, wt, &d, uid_step});
        else
#endif
            relax_slots<POL, STATS, FUSE, BIDIR>(p, v, c, W, fok, cd);
    }
}

// Relax the fused vertices (already deleted from / never entered Q, key known), 32 at a
// time from the top of the warp's stack; their relaxations may fuse more.  (The order
// matters: tried together with a lane-local relax for degree <= kArcs, a FIFO ring and
// slot-major pushes scanned 6-7x more arcs on grid4096 with Delta* = 2^17, 40-55 % slower.)
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void fuse_drain(const RunParams& p, Warp& W) {
    if (!FUSE) return;
    const int lane = lane_id();
    PROF_T0(tfd);
    while (W.fn > 0) {
#if SSSP_PROF
        W.prof[5]++;
#endif
        const int32_t cnt = W.fn < 32 ? W.fn : 32;
        __syncwarp();
        int32_t id = -1, dep = 0;
        uint64_t d = 0;
        if (lane < cnt) {
            id = W.fs()->fid[W.fn - cnt + lane];
            d = W.fs()->fd[W.fn - cnt + lane];
            dep = W.fs()->fdep[W.fn - cnt + lane];
        }
        __syncwarp();
        W.fn -= cnt;
        int32_t beg = 0, deg = 0;
        if (id >= 0) {
            beg = __ldg(p.off + id);
            deg = __ldg(p.off + id + 1) - beg;
        }
        // a fused hub goes back to Q instead (its arcs belong in chunks, not in one warp)
        bool back = false;
        const int32_t hub = id;
        if (id >= 0 && deg > kFuseMaxDeg) {
            const uint64_t old = atomicCAS((unsigned long long*)(p.dist + id), (unsigned long long)(d | kTop),
                                           (unsigned long long)d);
            back = old == (d | kTop) && admit<STATS>(old, d, W);  // else a later WriteMin re-inserted it
            id = -1;
            deg = 0;
        }
        wq_push1(W, back, hub);
        if (id >= 0) {
            if (p.ext_count) atomicAdd(p.ext_count + (p.ofno ? p.ofno[id] : id), 1);
            if (STATS) {
                W.acc.fused++;  // counted as inserted and extracted (the |Q| identity holds)
                W.acc.inserts++;
                W.acc.fused_edges += (uint64_t)deg;
            }
        }
        relax_vertices<POL, STATS, FUSE, BIDIR>(p, d, beg, deg, W, id, dep);
    }
    PROF_ADD(W, 4, tfd);
}

// Cut the heavy lanes' vertices into kChunk-arc descriptors (one reservation per warp).
__device__ __forceinline__ void emit_chunks(const Sharded<Desc>& CL, int shard, bool heavy, uint64_t d, int32_t beg,
                                            int32_t deg, RoundCnt* C, bool stats) {
    const uint32_t hm = __ballot_sync(kFull, heavy);
    if (!hm) return;
    const int lane = lane_id();
    const int32_t nch = heavy ? (deg + kChunk - 1) / kChunk : 0;
    const int32_t incl = warp_incl_scan(nch);
    const int32_t tot = __shfl_sync(kFull, incl, 31);
    const int32_t excl = incl - nch;
    if (stats && lane == 0) atomicAdd(&C->nheavy, __popc(hm));
    Desc *p0, *p1;
    int32_t fit, lim;
    reserve(CL, shard, tot, p0, fit, p1, lim);
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
        if (j < lim) {
            const int32_t k = (j - oe) * kChunk;
            st_desc(j < fit ? p0 + j : p1 + (j - fit), odd, ob + k, min(kChunk, od - k));
        }
    }
}

// --------------------------------------------------------------------- phase A
// Extract(theta) in two decoupled parts:
//  scan:  kEnt queue entries per lane per step (all id loads, then all key gathers in
//         flight); ids above theta are staged for the next queue, ids at or below it
//         are staged in the warp's take buffer;
//  batch: 32 staged ids at a time are deleted from Q (atomicOr, which returns the exact
//         key they relax with), their CSR rows read, heavy ones cut into chunks and the
//         light ones relaxed by the warp at once (live) or listed (snapshot).
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void take_batch(const RunParams& p, int32_t cnt, const Sharded<Desc>& CL, bool snap, Warp& W,
                                           uint64_t& fs, uint64_t& edges) {
    const int lane = lane_id();
    PROF_T0(tt);
    __syncwarp();
    int32_t id = lane < cnt ? W.st()->take[lane] : -1;
    // the CSR row is read alongside the delete (independent loads: one latency, not two);
    // the results are consumed by selects, not inside the branch, so they stay ahead of it
    int32_t beg = 0, end = 0;
    uint64_t old = kTop;
    if (id >= 0) {
        ld_row(p.off, id, beg, end);
        old = atom_or_u64(p.dist + id, kTop);  // delete from Q
    }
    const bool ok = !(old & kTop);  // else already deleted by another copy (safety net: not expected)
    const uint64_t d = old & kVal;
    const int32_t deg = ok ? end - beg : 0;
    beg = ok ? beg : 0;
    id = ok ? id : -1;
    {
        const uint32_t em = __ballot_sync(kFull, id >= 0);
#if !SSSP_FUSE_UNIT
        if (small_on(FUSE) && lane == 0) W.st()->ext += __popc(em);
#endif
    }
    if (id >= 0) {
        W.qdelta--;
        if (p.ext_count) atomicAdd(p.ext_count + (p.ofno ? p.ofno[id] : id), 1);
    }
    if (STATS && id >= 0) {
        fs += 1;
        edges += (uint64_t)deg;
    }
    const bool heavy = deg > kLight;
    const bool light = id >= 0 && deg > 0 && !heavy;
    emit_chunks(CL, W.shard(), heavy, d, beg, deg, W.C(), STATS);
    if (snap) {
        const int32_t ls = warp_append_slot(light, &W.C()->nlight);
        if (light) st_desc(p.light + ls, d, beg, deg);
    } else if (__any_sync(kFull, light)) {
        PROF_ADD(W, 1, tt);
        PROF_T0(tr);
        relax_vertices<POL, STATS, FUSE, BIDIR>(p, d, beg, light ? deg : 0, W, light ? id : -1);
        PROF_ADD(W, 2, tr);
        return;
    }
    PROF_ADD(W, 1, tt);
}

template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void phase_a(const RunParams& p, const Sharded<int32_t>& QC, const int64_t* qpref,
                                        const Sharded<Desc>& CL, uint64_t theta, bool snap, uint64_t& minrem, Warp& W,
                                        int32_t* tile_ctr) {
    const int lane = lane_id();
    const int64_t q = qpref[kSeg];
    const int64_t gw = warp_rank();
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t fs = 0, edges = 0;
    int32_t tn = 0;  // staged take ids (warp-uniform)
    // kEnt entries per lane only when every warp gets at least two such steps; small
    // queues are spread one entry per lane so that more warps share the round
    const int ent = q >= nwarps * (32 * kEnt) ? kEnt : 1;
    // Small queues: an equal contiguous share per warp (+-1 entry).  A round lasts as long
    // as its slowest warp; strided tiles left some warps with 3 tiles and others with 1,
    // and contiguous ids (appended together) keep a warp's fusion local.  Large queues:
    // strided tiles, since ids appended together carry correlated work (R-MAT hubs).
    const bool contig = q < (int64_t)kContigTiles * 32 * nwarps;
    const int64_t lo = contig ? gw * q / nwarps : gw * (32 * ent);
    const int64_t hi = contig ? (gw + 1) * q / nwarps : q;
    const int64_t stride = contig ? 32 * ent : nwarps * (32 * ent);
    // Dynamic tiles (kernels without fusion, queues of >= one 32-id tile per warp): the queue
    // is cut into 32*ent-id tiles dealt to the CTAs round-robin (CTA c owns tiles c,
    // c + grid, ...: correlated neighbours land on different SMs), and each CTA's warps
    // take its tiles from a shared-memory counter (no warp idles while its CTA has work).
    // With fusion, every warp keeps its own thin share: there each warp seeds its own
    // local search (dynamic tiles left most warps idle and took grid4096 from 932 to
    // 4,422 rounds).
    const bool dyn = !FUSE && q >= 32 * nwarps;
    for (int64_t it = 0;; it++) {
        int64_t base, lim;
        if (dyn) {
            int32_t k = 0;
            if (lane == 0) k = atomicAdd(tile_ctr, 1);
            k = __shfl_sync(kFull, k, 0);
            base = ((int64_t)k * gridDim.x + blockIdx.x) * (32 * ent);
            if (base >= q) break;
            lim = q;
        } else {
            base = lo + it * stride;
            if (base >= hi) break;
            lim = hi;
        }
        PROF_T0(ts);
        int32_t id[kEnt];
        uint64_t val[kEnt];
        const int sg = seg_of(qpref, base);  // warp-uniform
#pragma unroll
        for (int e = 0; e < kEnt; e++) {
            const int64_t i = base + e * 32 + lane;
            id[e] = -1;
            if (e < ent && i < lim) {
                int s = sg;
                while (qpref[s + 1] <= i) s++;
                id[e] = ld_cg_i32(QC.seg(s) + (i - qpref[s]));
            }
        }
#pragma unroll
        for (int e = 0; e < kEnt; e++) val[e] = id[e] >= 0 ? (ld_cg_u64(p.dist + id[e]) & kVal) : kVal;
#pragma unroll
        for (int e = 0; e < kEnt; e++) {
            const bool take = id[e] >= 0 && val[e] <= theta;
            const bool rem = id[e] >= 0 && !take;
            wq_push1(W, rem && val[e] <= W.split, id[e]);  // above the split: stays in Q as a far member
            if (uses_min(POL) && rem) minrem = val[e] < minrem ? val[e] : minrem;
            const uint32_t tm = __ballot_sync(kFull, take);
            if (take) W.st()->take[tn + __popc(tm & lanemask_lt())] = id[e];
            tn += __popc(tm);
        }
        PROF_ADD(W, 0, ts);
        int32_t done = 0;
        while (tn - done >= 32) {
            if (done) {  // move the next 32 to the front (take_batch reads take[0..32))
                __syncwarp();
                const int32_t x = W.st()->take[done + lane];
                __syncwarp();
                W.st()->take[lane] = x;
            }
            take_batch<POL, STATS, FUSE, BIDIR>(p, 32, CL, snap, W, fs, edges);
            done += 32;
        }
        if (done) {  // keep the remainder (< 32) at the front
            __syncwarp();
            const bool mv = lane < tn - done;
            int32_t x = 0;
            if (mv) x = W.st()->take[done + lane];
            __syncwarp();
            if (mv) W.st()->take[lane] = x;
            tn -= done;
        }
    }
    if (tn) take_batch<POL, STATS, FUSE, BIDIR>(p, tn, CL, snap, W, fs, edges);
    fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
    if (STATS) {
        fs = warp_sum(fs);
        edges = warp_sum(edges);
        if (lane == 0 && fs) atomicAdd(&W.C()->fsize, (unsigned long long)fs);
        if (lane == 0 && edges) atomicAdd(&W.C()->edges, (unsigned long long)edges);
    }
}

// --------------------------------------------------------------------- phase B
#ifndef SSSP_DYN_B
#define SSSP_DYN_B 0
#endif
#ifndef SSSP_NEXT_SMEM
#define SSSP_NEXT_SMEM 1  // static phase-B order: next descriptor by cp.async into shared memory
#endif
// dyn_ctr != nullptr (SSSP_DYN_B, grid rounds): CTA c owns items c, c + grid, c + 2 grid, ...
// and its warps take the next one from a shared-memory counter (no warp idles while its CTA
// has items left); else warp gw strides over all items by nwarps.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void phase_b(const RunParams& p, const Sharded<Desc>& CL, const int64_t* cpref, int32_t nl,
                                        Warp& W, int64_t gw, int64_t nwarps, int32_t* dyn_ctr = nullptr) {
    const int lane = lane_id();
    if (SSSP_DYN_B && dyn_ctr) {
        const int64_t nc = cpref[kSeg];
        int sh = 0;
        auto take = [&]() {
            int32_t k = 0;
            if (lane == 0) k = atomicAdd(dyn_ctr, 1);
            return (int64_t)__shfl_sync(kFull, k, 0) * gridDim.x + blockIdx.x;
        };
        // the next item's descriptor is prefetched by lane 0 with a 16-byte cp.async into the
        // warp's stage (held in registers across the relax it spilled: 8 local-memory
        // instructions per chunk, 29 M per rmat24 run)
        Desc* nd = W.st()->nd;
        auto prefetch = [&](int64_t i, int slot) {
            while (sh < kShards && cpref[sh + 1] <= i) sh++;  // a warp's items only increase
            if (lane == 0) cp_async16(nd + slot, CL.seg(sh) + (i - cpref[sh]));
        };
        int64_t item = take();
        int cur = 0;
        if (item < nc) prefetch(item, 0);
        while (item < nc) {
            cp_async_wait_all();
            __syncwarp();
            const Desc e = nd[cur];
            item = take();
            if (item < nc) prefetch(item, cur ^ 1);
            cur ^= 1;
            relax_chunk<POL, STATS, FUSE, BIDIR>(p, e.d, e.beg, e.len, W);
            if (FUSE && W.fn > kFBuf - 32 * kArcs) fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
        }
        fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
        return;
    }
    const int64_t nb = ((int64_t)nl + 31) / 32;
    const int64_t nc = cpref[kSeg];
    const int64_t total = nb + nc;
    int sh = 0;  // SSSP_SEG_HINT: segment of the last descriptor read (a warp's items only increase)
#if SSSP_NEXT_SMEM
    // the next chunk descriptor is prefetched into the warp's stage by a 16-byte cp.async
    // (see the dynamic path above; rmat24 rho 2^18 -6.5 %, Delta* -6 % with the dynamic path)
    Desc* nd = W.st()->nd;
    int cur = 0;
    auto prefetch = [&](int64_t i, int slot) {  // i-th descriptor of the concatenated segments
        if (SSSP_SEG_HINT) {
            while (sh < kShards && cpref[sh + 1] <= i) sh++;
        } else {
            sh = seg_of(cpref, i);
        }
        if (lane == 0) cp_async16(nd + slot, CL.seg(sh) + (i - cpref[sh]));
    };
    int64_t item = gw;
    if (item >= nb && item < total) prefetch(item - nb, 0);
    for (; item < total; item += nwarps) {
        if (item < nb) {
            const int64_t j = item * 32 + lane;
            Desc e;
            if (j < nl) {
                e = ld_desc(p.light + j);
            } else {
                e.d = 0;
                e.beg = 0;
                e.len = 0;
            }
            relax_vertices<POL, STATS, FUSE, BIDIR>(p, e.d, e.beg, e.len, W);
            if (item + nwarps >= nb && item + nwarps < total) prefetch(item + nwarps - nb, cur);
        } else {
            cp_async_wait_all();
            __syncwarp();
            const Desc e = nd[cur];
            if (item + nwarps < total) prefetch(item + nwarps - nb, cur ^ 1);
            cur ^= 1;
            relax_chunk<POL, STATS, FUSE, BIDIR>(p, e.d, e.beg, e.len, W);
            if (FUSE && W.fn > kFBuf - 32 * kArcs) fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
        }
    }
#else
    // (Bellman-Ford's unit keeps the descriptor in registers: +4.6 % on rmat24 with cp.async)
    auto chunk_at = [&](int64_t i) {  // i-th descriptor of the concatenated segments
        if (SSSP_SEG_HINT) {
            while (sh < kShards && cpref[sh + 1] <= i) sh++;
        } else {
            sh = seg_of(cpref, i);
        }
        return ld_desc(CL.seg(sh) + (i - cpref[sh]));
    };
    int64_t item = gw;
    Desc nxt;
    if (item >= nb && item < total) nxt = chunk_at(item - nb);
    for (; item < total; item += nwarps) {
        if (item < nb) {
            const int64_t j = item * 32 + lane;
            Desc e;
            if (j < nl) {
                e = ld_desc(p.light + j);
            } else {
                e.d = 0;
                e.beg = 0;
                e.len = 0;
            }
            relax_vertices<POL, STATS, FUSE, BIDIR>(p, e.d, e.beg, e.len, W);
            if (item + nwarps >= nb && item + nwarps < total) nxt = chunk_at(item + nwarps - nb);
        } else {
            const Desc e = nxt;
            if (item + nwarps < total) nxt = chunk_at(item + nwarps - nb);  // prefetch
            relax_chunk<POL, STATS, FUSE, BIDIR>(p, e.d, e.beg, e.len, W);
            if (FUSE && W.fn > kFBuf - 32 * kArcs) fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
        }
    }
#endif
    fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
}

template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void flush_acc(const RunParams& p, int64_t r, Warp& W) {
    drain_pending<POL, STATS, FUSE, BIDIR>(p, W);  // deferred WriteMins before the phase ends
    wq_flush(W);
    const int64_t dq = warp_sum(W.qdelta);
    if (lane_id() == 0 && dq) atomicAdd((unsigned long long*)(p.cta_delta + (r % 3) * kMaxCtas + blockIdx.x),
                                        (unsigned long long)dq);
    W.qdelta = 0;
#if !SSSP_FUSE_UNIT
    if (small_on(FUSE) && lane_id() == 0 && W.st()->ext) {
        atomicAdd(p.cta_ext + (r % 3) * kMaxCtas + blockIdx.x, W.st()->ext);
        W.st()->ext = 0;
    }
#endif
    if (STATS) {
        const uint32_t s = warp_sum(W.acc.succ), ins = warp_sum(W.acc.inserts), fu = warp_sum(W.acc.fused);
        const uint64_t fe = warp_sum(W.acc.fused_edges);
        if (lane_id() == 0 && s) atomicAdd(&W.C()->succ, (unsigned long long)s);
        if (lane_id() == 0 && ins) atomicAdd(&W.C()->inserts, (unsigned long long)ins);
        if (lane_id() == 0 && fu) atomicAdd(&W.C()->fsize, (unsigned long long)fu);
        if (lane_id() == 0 && fu) atomicAdd(&W.C()->fused, (unsigned long long)fu);
        if (lane_id() == 0 && fe) atomicAdd(&W.C()->edges, (unsigned long long)fe);
    }
    W.acc.succ = 0;
    W.acc.inserts = 0;
    W.acc.fused = 0;
    W.acc.fused_edges = 0;
}

// --------------------------------------------------------------------- ExtDist for rho
struct SmemKey {
    const uint64_t* a;
    __device__ uint64_t operator()(int64_t i) const { return a[i]; }
};
struct QueueVal {  // value of the i-th queued id (flag bit masked off), read through L2
    Sharded<int32_t> Q;
    const int64_t* pref;
    const uint64_t* dist;
    __device__ uint64_t operator()(int64_t i) const {
        const int s = seg_of(pref, i);
        return ld_cg_u64(dist + ld_cg_i32(Q.seg(s) + (i - pref[s]))) & kVal;
    }
};

__device__ __forceinline__ uint64_t sample_index(uint64_t seed, int64_t round, uint64_t j, uint64_t q) {
    return splitmix64(seed ^ splitmix64(((uint64_t)round << 32) | j)) % q;
}

// k-th smallest (1-based) of s <= blockDim keys in shared memory by rank counting:
// the key x with #{< x} < k <= #{<= x}.  P = 4, 2 or 1 adjacent lanes share a key (as many as the
// CTA has threads for) and count interleaved slices of the keys, combined by shuffles: the
// select runs on every CTA at every round top, so its length is round latency (s = 256 on
// 1,024 threads: 64 iterations per thread instead of 256).  Two barriers.
__device__ __forceinline__ uint64_t cta_kth_by_rank(const uint64_t* keys, int s, uint64_t k, SelectSmem& sm) {
    const int tid = threadIdx.x;
    const int lg = s * 4 <= (int)blockDim.x ? 2 : (s * 2 <= (int)blockDim.x ? 1 : 0);  // log2 P (CTA-uniform)
    const int P = 1 << lg, ki = tid >> lg, part = tid & (P - 1);
    const bool on = ki < s;
    const uint64_t x = on ? keys[ki] : 0;
    uint32_t lt = 0, le = 0;
    if (on) {
        int j = part;
        for (; j + 7 * P < s; j += 8 * P) {  // 8 independent loads in flight
            uint64_t y[8];
#pragma unroll
            for (int u = 0; u < 8; u++) y[u] = keys[j + u * P];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                lt += y[u] < x;
                le += y[u] <= x;
            }
        }
        for (; j < s; j += P) {
            const uint64_t y = keys[j];
            lt += y < x;
            le += y <= x;
        }
    }
    if (lg >= 1) {  // (whole warps take this branch: lg is CTA-uniform)
        lt += __shfl_xor_sync(kFull, lt, 1);
        le += __shfl_xor_sync(kFull, le, 1);
    }
    if (lg >= 2) {
        lt += __shfl_xor_sync(kFull, lt, 2);
        le += __shfl_xor_sync(kFull, le, 2);
    }
    if (on && part == 0 && lt < k && k <= le) sm.bcast[0] = x;  // every writer writes the same value
    __syncthreads();
    const uint64_t th = sm.bcast[0];
    __syncthreads();
    return th;
}

// --------------------------------------------------------------------- near/far queue
// The queue array holds only the NEAR members of Q (key <= split); FAR members (key >
// split) are implicit: their flag bit says "in Q" and nothing else lists them.  When the
// near part runs low, a coalesced dense pass over delta moves the FAR keys in (split,
// split'] into the queue (DESIGN.md §5 "near/far").  Rounds then rescan ~kNearK rounds
// of work instead of all of Q.

// Dense pass: append every far member with value in (lo, hi] to the list L (staged).
__device__ __forceinline__ void far_to_near(const RunParams& p, const Sharded<int32_t>& L, uint64_t lo, uint64_t hi,
                                            Warp& W) {
    const int lane = lane_id();
    const Sharded<int32_t> saved = W.swap_qnext(L);
    const int64_t gw = warp_rank();
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int kV = 8;  // keys in flight per lane per step (12 / 16: +0 to +1.7 %, registers)
    for (int64_t base = gw * (32 * kV); base < p.n; base += nwarps * (32 * kV)) {
        uint64_t x[kV];
#pragma unroll
        for (int t = 0; t < kV; t++) {
            const int64_t v = base + t * 32 + lane;
            x[t] = v < p.n ? __ldcg((const unsigned long long*)(p.dist + v)) : kInf;
        }
#pragma unroll
        for (int t = 0; t < kV; t++) {
            const uint64_t val = x[t] & kVal;
            wq_push1(W, !(x[t] & kTop) && val > lo && val <= hi, (int32_t)(base + t * 32 + lane));
        }
    }
    wq_flush(W);
    W.swap_qnext(saved);
}

// CTA-0 estimate of the value below which about `want` far members lie: rejection-sample
// vertices, keep the far ones, take the matching order statistic (kInf if none seen).
static __device__ __forceinline__ uint64_t far_quantile(const RunParams& p, uint64_t split, int64_t far, int64_t want, int64_t r,
                                 uint64_t* keys, SelectSmem& sm, int32_t* cnt) {
    if (threadIdx.x == 0) *cnt = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < kFarSamples; j += blockDim.x) {
        const uint64_t v = splitmix64(p.seed ^ 0xF00DF00DF00DULL ^ splitmix64(((uint64_t)r << 32) | (uint64_t)j)) %
                           (uint64_t)p.n;
        const uint64_t x = __ldcg((const unsigned long long*)(p.dist + v));
        if (!(x & kTop) && (x & kVal) > split) keys[atomicAdd(cnt, 1)] = x & kVal;
    }
    __syncthreads();
    const int32_t h = *cnt;
    if (h == 0) return kInf;
    uint64_t k = (uint64_t)(((double)want / (double)far) * h) + 1;
    k = k > (uint64_t)h ? (uint64_t)h : k;
    return h <= kRankSelect ? cta_kth_by_rank(keys, h, k, sm) : cta_kth_smallest(SmemKey{keys}, h, k, sm);
}

// --------------------------------------------------------------------- small-frontier rounds
struct SmallKey {  // key of the i-th id of a shared-memory queue
    const int32_t* q;
    const uint64_t* dist;
    __device__ uint64_t operator()(int64_t i) const { return ld_cg_u64(dist + q[i]) & kVal; }
};
__device__ __forceinline__ uint64_t atom_and_u64(uint64_t* p, uint64_t x) {
    uint64_t old;
    asm volatile("atom.global.and.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(x) : "memory");
    return old;
}
// theta_i = i * Delta, skipping empty steps (reading R2), saturating
__device__ __forceinline__ uint64_t delta_next(uint64_t theta_prev, uint64_t minq, uint64_t D) {
    const uint64_t x = theta_prev > kInf - D ? kInf : theta_prev + D;
    const uint64_t y = (minq / D + (minq % D != 0)) * D;
    return x > y ? x : y;
}

#if !SSSP_FUSE_UNIT
// Rounds r, r+1, ... of Alg. 1 run by CTA 0 alone (all 1024 threads call it), starting from
// Q_r (|Q_r| = qtot <= kSmallQ ids, all listed in the grid's queue QC0 / qpref0).  Each round:
//   ExtDist per policy (as the grid computes it, over all of Q);
//   Extract: every queued id is deleted by atomicOr (which returns its key) and its CSR row
//            read alongside; ids above theta are put back (atomicAnd) and kept;   CTA barrier
//   if the frontier has more than kSmallArcs arcs: undo the round and hand it to the grid;
//   Relax: light vertices by the warp that holds them, heavy ones as chunk descriptors that
//          all 32 warps stride over (phase_b); WriteMins append to Q_{r+1} in shared memory;
//          fusion as in the grid's live rounds.                               CTA barrier
// Every round extracts before it relaxes, with the keys Extract returned: the LaB-PQ's
// exclusive Extract, i.e. the grid's snapshot rounds.  Returns when Q is empty,
// |Q| > kSmallQ, or a frontier is too large; Q is then written back in the grid's layout and
// the resume state to ctrl (sm_*); the caller releases the other CTAs.
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__device__ __forceinline__ void small_rounds(const RunParams& p, int64_t r, int64_t qtot, uint64_t theta_prev, int warm, uint64_t minq,
                  const Sharded<int32_t> QC0, const int64_t* qpref0, int64_t* cpref, uint64_t* red) {
    // (inlined outside the grid's round loop; a __noinline__ version, which must read the
    // parameters through a global copy, was 4-20 % slower per small round)
    constexpr int kE = kSmallQ / kBlock;  // queue entries per thread
    const int tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    uint64_t* s_keys = (uint64_t*)(sssp_dyn_smem + kWarps * sizeof(WarpStage));
    SelectSmem& sm = *(SelectSmem*)(s_keys + kSmemSamples);
    Warp W;  // this warp's state for the small rounds (the grid's is empty between rounds)
    W.init();
    W.qn = W.fn = W.pn = 0;
    W.qdelta = 0;
#if SSSP_PROF
    for (int i = 0; i < kProf; i++) W.prof[i] = 0;
#endif
    Ctrl* ctrl = p.ctrl;
    const bool snap = (p.flags & SSSP_RUN_SNAPSHOT) != 0;
    const int64_t qcap = p.qcap;
    for (int64_t i = tid; i < qtot; i += blockDim.x) {
        const int sg = seg_of(qpref0, i);
        s_small.q[0][i] = ld_cg_i32(QC0.seg(sg) + (i - qpref0[sg]));
    }
    if (tid == 0) {  // (q[k] is Q of the rounds r0 + k, r0 + k + 2, ...)
        s_small.on = 1;
        s_small.qcnt[0] = (int32_t)qtot;
        s_small.qcnt[1] = 0;
        s_small.qcap = qcap;
        s_small.gq[0] = p.qbuf[r & 1];
        s_small.gq[1] = p.qbuf[(r + 1) & 1];
        for (int k = 0; k < 2; k++) {
            s_small.arcs[k] = 0;
            s_small.heavy[k] = 0;
            s_small.ext[k] = 0;
        }
    }
    W.split = kInf;
    W.fuse_theta = 0;
    int cur = 0;
    int end = 0;  // 1: Q empty / rounds exceeded; 2: Q_r handed to the grid
    int32_t last_ext = 0;  // extractions of the last round run here (the grid's entry test)
    __syncthreads();
    for (;;) {
        if (r > p.max_rounds) {
            if (tid == 0) ctrl->status = SSSP_ERR_ROUNDS;
            end = 1;
            break;
        }
        RoundCnt* C = &ctrl->cnt[r % 3];
        uint64_t t0 = 0, t1 = 0, t2 = 0;
        if (STATS && tid == 0) t0 = globaltimer();
        const int32_t* q = s_small.q[cur];
        const int32_t qn = (int32_t)qtot;
        const uint64_t theta_prev0 = theta_prev;  // (restored if the round is handed to the grid)
        const int warm0 = warm;
        // ---- ExtDist (Table tab:framework), over all of Q
        uint64_t theta;
        if (POL == SSSP_BELLMAN_FORD) {
            theta = kInf;
        } else if (POL == SSSP_DIJKSTRA) {
            theta = minq;
        } else if (POL == SSSP_DELTA_STEPPING && r > 1 && minq <= theta_prev) {
            theta = theta_prev;  // FinishCheck failed (R19)
        } else if (POL == SSSP_DELTA || POL == SSSP_DELTA_STEPPING) {
            theta = delta_next(theta_prev, minq, p.param);
            theta_prev = theta;
        } else {  // rho
            uint64_t rho = p.param;
            if (!(p.flags & SSSP_RUN_NO_WARMUP) && (uint64_t)qtot > rho && warm < 2) {
                warm++;
                rho = rho / 10 ? rho / 10 : 1;  // reading R7
            }
            if ((uint64_t)qtot <= rho) {
                theta = kInf;
            } else if (p.flags & SSSP_RUN_RHO_EXACT) {
                theta = cta_kth_smallest(SmallKey{q, p.dist}, qtot, rho, sm);
            } else {
                const uint64_t sc = sample_count((uint64_t)qtot, rho);
                uint64_t* keys = sc <= (uint64_t)kSmemSamples ? s_keys : p.samples;
                for (uint64_t j = tid; j < sc; j += blockDim.x)
                    keys[j] = ld_cg_u64(p.dist + q[sample_index(p.seed, r, j, (uint64_t)qtot)]) & kVal;
                __syncthreads();
                uint64_t k = (rho * sc + (uint64_t)qtot - 1) / (uint64_t)qtot;
                k = k < 1 ? 1 : (k > sc ? sc : k);
                theta = sc <= (uint64_t)kRankSelect ? cta_kth_by_rank(keys, (int)sc, k, sm)
                                                    : cta_kth_smallest(ArrayKey{keys}, (int64_t)sc, k, sm);
            }
        }
        if (STATS && tid == 0) t1 = globaltimer();
        const int nxt = cur ^ 1;
        if (tid < 2 * kSeg)  // counters of slot (r+1)%3 (the chunk list of round r+1)
            p.counters[((int64_t)(((r + 1) % 3) * 2) * kSeg + tid) * kCntStride] = 0;
        if (tid == 0) reset_cnt(&ctrl->cnt[(r + 1) % 3]);
        if (lane == 0) W.st()->snxt = nxt;
        W.fuse_theta = (FUSE && !snap) ? theta : 0;
        // (no barrier: every shared scalar this round uses was reset during the previous one)
        // ---- Extract(theta): delete every queued id, keep those above theta
        int32_t id[kE], beg[kE], deg[kE];
        uint64_t d[kE];
        bool keep[kE];
        uint64_t minrem = kInf;
        unsigned long long arcs = 0;
#pragma unroll
        for (int e = 0; e < kE; e++) {
            const int i = e * kBlock + tid;
            id[e] = -1;
            deg[e] = 0;
            beg[e] = 0;
            d[e] = 0;
            keep[e] = false;
            if (i < qn) {
                const int32_t v = q[i];
                int32_t b, en;
                ld_row(p.off, v, b, en);
                const uint64_t old = atom_or_u64(p.dist + v, kTop);
                const uint64_t key = old & kVal;
                if (!(old & kTop)) {  // (every listed id is in Q; a deleted one is skipped)
                    if (key <= theta) {
                        id[e] = v;
                        d[e] = key;
                        beg[e] = b;
                        deg[e] = en - b;
                        arcs += (unsigned long long)(en - b);
                    } else {
                        atom_and_u64(p.dist + v, ~kTop);  // back into Q (no WriteMin runs yet)
                        minrem = key < minrem ? key : minrem;
                        keep[e] = true;
                    }
                }
            }
        }
        arcs = warp_sum(arcs);
        if (lane == 0 && arcs) atomicAdd(&s_small.arcs[r & 1], arcs);
        __syncthreads();
        if (s_small.arcs[r & 1] > (unsigned long long)kSmallArcs) {
            // too much work for one SM: undo the deletions and hand round r to the grid
#pragma unroll
            for (int e = 0; e < kE; e++)
                if (id[e] >= 0) atom_and_u64(p.dist + id[e], ~kTop);
            theta_prev = theta_prev0;
            warm = warm0;
            end = 2;
            break;
        }
        if (tid == 0) {  // the next round's scalars (q[cur] is read no more this round)
            s_small.qcnt[cur] = 0;
            s_small.arcs[(r + 1) & 1] = 0;
            s_small.heavy[(r + 1) & 1] = 0;
            s_small.ext[(r + 1) & 1] = 0;
        }
        // kept ids go to Q_{r+1} first (in queue order)
#pragma unroll
        for (int e = 0; e < kE; e++) wq_push1(W, keep[e], keep[e] ? q[e * kBlock + tid] : -1);
        int64_t fs = 0;
#pragma unroll
        for (int e = 0; e < kE; e++) {
            const uint32_t em = __ballot_sync(kFull, id[e] >= 0);
            if (lane == 0) W.st()->ext += __popc(em);
        }
#pragma unroll
        for (int e = 0; e < kE; e++)
            if (id[e] >= 0) {
                fs++;
                if (p.ext_count) atomicAdd(p.ext_count + (p.ofno ? p.ofno[id[e]] : id[e]), 1);
            }
        if (STATS) {
            fs = warp_sum(fs);
            const unsigned long long a = arcs;
            if (lane == 0 && fs) atomicAdd(&C->fsize, (unsigned long long)fs);
            if (lane == 0 && a) atomicAdd(&C->edges, a);
        }
        // ---- Relax (with the keys Extract returned)
        W.fbudget = p.fuse_budget;
        const Sharded<Desc> CL = chunks_of(p, r);
#pragma unroll
        for (int e = 0; e < kE; e++) {
            const bool heavy = deg[e] > kLight;
            const bool light = id[e] >= 0 && deg[e] > 0 && !heavy;
            if (__any_sync(kFull, heavy)) {
                if (lane == 0) s_small.heavy[r & 1] = 1;
                emit_chunks(CL, W.shard(), heavy, d[e], beg[e], deg[e], C, STATS);
            }
            if (__any_sync(kFull, light))
                relax_vertices<POL, STATS, FUSE, BIDIR>(p, d[e], beg[e], light ? deg[e] : 0, W, light ? id[e] : -1);
        }
        fuse_drain<POL, STATS, FUSE, BIDIR>(p, W);
        __syncthreads();
        if (s_small.heavy[r & 1]) {  // heavy vertices: all warps of the CTA stride over their chunks
            load_prefix(CL, cpref);
            phase_b<POL, STATS, FUSE, BIDIR>(p, CL, cpref, 0, W, wid, kWarps);
        }
        drain_pending<POL, STATS, FUSE, BIDIR>(p, W);
        wq_flush(W);
        if (STATS) {
            const uint32_t sc = warp_sum(W.acc.succ), ins = warp_sum(W.acc.inserts), fu = warp_sum(W.acc.fused);
            const uint64_t fe = warp_sum(W.acc.fused_edges);
            if (lane == 0 && sc) atomicAdd(&C->succ, (unsigned long long)sc);
            if (lane == 0 && ins) atomicAdd(&C->inserts, (unsigned long long)ins);
            if (lane == 0 && fu) atomicAdd(&C->fsize, (unsigned long long)fu);
            if (lane == 0 && fu) atomicAdd(&C->fused, (unsigned long long)fu);
            if (lane == 0 && fe) atomicAdd(&C->edges, (unsigned long long)fe);
            W.acc.succ = W.acc.inserts = W.acc.fused = 0;
            W.acc.fused_edges = 0;
        }
        // min_Q delta of Q_{r+1}: kept keys and successful WriteMins (Delta* / Dijkstra)
        if (uses_min(POL)) {
            const uint64_t mn = warp_min_u64(minrem < W.acc.minsucc ? minrem : W.acc.minsucc);
            if (lane == 0) red[wid] = mn;
            W.acc.minsucc = kInf;
        }
        W.qdelta = 0;
        if (lane == 0 && W.st()->ext) {
            atomicAdd(&s_small.ext[r & 1], W.st()->ext);
            W.st()->ext = 0;
        }
        __syncthreads();
        const int32_t ext = s_small.ext[r & 1];
        if (uses_min(POL)) {
            uint64_t mn = kInf;
            static_assert(kWarps <= 32, "one per-warp minimum per lane");
            mn = warp_min_u64(lane < kWarps ? red[lane] : kInf);  // every warp reduces the warp minima itself
            minq = mn;
        }
        const int64_t qnext = s_small.qcnt[nxt];
        if (STATS && tid == 0) {
            t2 = globaltimer();
            const int64_t f = (int64_t)C->fsize;
            if (p.trace && r - 1 < p.trace_cap) {
                sssp_round* t = p.trace + (r - 1);
                memset(t, 0, sizeof(*t));
                t->qsize = qtot;
                t->fsize = f;
                t->edges = (int64_t)C->edges;
                t->inserts = (int64_t)C->inserts;
                t->succ = (int64_t)C->succ;
                t->theta = theta;
                t->nheavy = (int64_t)C->nheavy;
                t->t_theta_ns = (int64_t)(t1 - t0);
                t->t_extract_ns = (int64_t)(t2 - t1);
                t->qnear = qtot;
                t->fused = (int64_t)C->fused;
                t->small = 1;
            }
            ctrl->tot_extracted += f;
            ctrl->tot_edges += (int64_t)C->edges;
            ctrl->tot_succ += (int64_t)C->succ;
            ctrl->tot_inserts += (int64_t)C->inserts;
            ctrl->tot_qscan += qtot;
            ctrl->max_q = qtot > ctrl->max_q ? qtot : ctrl->max_q;
            ctrl->max_f = f > ctrl->max_f ? f : ctrl->max_f;
            ctrl->sm_rounds++;
        }
        r++;
        qtot = qnext;
        cur = nxt;
        if (qtot == 0) {
            end = 1;
            break;
        }
        if (qtot > kSmallQ || ext > 2 * kSmallF) {
            last_ext = ext;
            end = 2;
            break;
        }
    }
    // ---- hand back: Q_r in the grid's layout (flat: shard-0 segment, then the spill segment)
    if (end == 2) {
        int32_t* gq = p.qbuf[r & 1];
        const int64_t ns = qtot < kSmallQ ? qtot : kSmallQ;  // the rest is in gq already
        for (int64_t i = tid; i < ns; i += blockDim.x) *flat_slot(gq, qcap, i) = s_small.q[cur][i];
        // queue counts of Q_r: slot (r+2)%3, list 0
        int32_t* qc = p.counters + (int64_t)((((r + 2) % 3) * 2) * kSeg) * kCntStride;
        if (tid < kSeg)
            qc[tid * kCntStride] = tid == 0 ? (int32_t)qtot : (tid == kShards ? (int32_t)(qtot > qcap ? qtot - qcap : 0) : 0);
        // min_Q of Q_r and the extractions of round r-1 as per-CTA values of round r-1
        for (int i = tid; i < (int)gridDim.x; i += blockDim.x) {
            p.cta_min[((r + 2) % 3) * kMaxCtas + i] = i == 0 ? minq : kInf;
            p.cta_ext[((r + 2) % 3) * kMaxCtas + i] = i == 0 ? last_ext : 0;
        }
    }
    if (tid == 0) {
        s_small.on = 0;
        ctrl->sm_end = end == 1;
        ctrl->sm_r = r;
        ctrl->sm_qtot = qtot;
        ctrl->sm_theta_prev = theta_prev;
        ctrl->sm_warm = warm;
    }
    __syncthreads();
}

#endif  // !SSSP_FUSE_UNIT

// --------------------------------------------------------------------- the round loop
template <int POL, bool STATS, bool FUSE, bool BIDIR>
__global__ void __launch_bounds__(kBlock, kMinBlocks) sssp_round_loop(RunParams p) {
    unsigned char* smem_raw = sssp_dyn_smem;
    uint64_t* s_keys = (uint64_t*)(smem_raw + kWarps * sizeof(WarpStage));  // [kSmemSamples]
    SelectSmem& sm = *(SelectSmem*)(s_keys + kSmemSamples);
    __shared__ int64_t qpref[kSeg + 1];  // segment prefix of Q_r's near part
    __shared__ int64_t cpref[kSeg + 1];  // segment prefix of the round's chunk list
    __shared__ uint64_t bc_u[3];         // min_Q (Delta / Dijkstra), CTA-0 theta, CTA-0 split
    __shared__ int64_t bc_dq;
    __shared__ int32_t bc_ext;           // extractions of the previous round (small-round entry test)
    __shared__ int32_t bc_nl, bc_cnt;
    __shared__ int32_t tile_ctr[4];      // phase-A [0, 1] and phase-B [2, 3] item counters, by round parity
    __shared__ uint64_t red[kWarps];
#ifndef SSSP_BAL
#define SSSP_BAL 0
#endif
#if SSSP_BAL
    __shared__ unsigned long long bal[2];
    if (threadIdx.x == 0) bal[0] = bal[1] = 0;
#endif
    Ctrl* ctrl = p.ctrl;
    Warp W;
    W.init();
    W.qn = 0;
    W.fn = 0;
    W.pn = 0;
#if !SSSP_FUSE_UNIT
    if (lane_id() == 0) W.st()->ext = 0;
#endif
    if (threadIdx.x == 0) tile_ctr[0] = tile_ctr[1] = tile_ctr[2] = tile_ctr[3] = 0;
    W.qdelta = 0;
#if SSSP_PROF
    for (int i = 0; i < kProf; i++) W.prof[i] = 0;
#endif
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;

    // Alg. 1 lines 1-2: delta[.] = +inf (not in Q), delta[s] = 0 (in Q), Q_1 = {s}
    // the source in run ids (an isolated source of a compacted graph lies past p.n: it is
    // extracted in round 1 and relaxes nothing)
    const int32_t src = p.nofo ? p.nofo[p.source] : p.source;
    // cold loop state of the small-frontier hand-over, kept in shared memory (not registers)
    __shared__ struct {
        int32_t epoch;    // small-frontier hand-backs seen
        int32_t resumed;  // this round follows small rounds: qtot is CTA 0's count
        int32_t cool;     // the last small attempt handed its first round back: the grid runs it
        int32_t src_deg;  // round 1's frontier arcs
    } ls;
    if (threadIdx.x == 0) {
        ls.epoch = ls.resumed = ls.cool = 0;
        ls.src_deg = __ldg(p.off + src + 1) - __ldg(p.off + src);
    }
    for (int64_t i = gtid; i < p.n; i += gsize) p.dist[i] = (i == src) ? 0ull : kInf;
    if (gtid == 0 && src >= p.n) p.dist[src] = 0;
    if (p.ext_count)
        for (int64_t i = gtid; i < (p.nofo ? p.n_out : p.n); i += gsize) p.ext_count[i] = 0;
    for (int64_t i = gtid; i < 3 * 2 * kSeg; i += gsize) p.counters[i * kCntStride] = 0;
    for (int64_t i = gtid; i < 3 * kMaxCtas; i += gsize) {
        p.cta_min[i] = kInf;
        p.cta_delta[i] = 0;
        p.cta_ext[i] = 0;
    }
    if (gtid == 0) {
        p.qbuf[1][0] = src;  // Q_1 lives in qbuf[1], shard 0
        for (int c = 0; c < 3; c++) reset_cnt(&ctrl->cnt[c]);
        ctrl->status = 0;
        ctrl->rounds = 0;
        ctrl->tot_extracted = ctrl->tot_edges = ctrl->tot_succ = ctrl->tot_inserts = 0;
        ctrl->tot_qscan = ctrl->max_q = ctrl->max_f = 0;
        ctrl->tot_dense = 0;
        ctrl->sm_epoch = 0;
        ctrl->sm_rounds = 0;
    }
#if !SSSP_FUSE_UNIT
    if (threadIdx.x == 0) s_small.on = 0;
#endif
    grid_sync();
    if (gtid == 0) {
        p.counters[0] = 1;  // |Q_1| = 1 (slot 0, queue list, shard 0)
        p.cta_min[0] = 0;   // min_Q delta = delta[s] = 0
    }
    grid_sync();

    // near/far queue for rho only (Delta* / BF / Dijkstra keep split = +inf: all of Q listed)
    const bool nearfar = POL == SSSP_RHO && !(p.flags & SSSP_RUN_NO_NEARFAR);
    uint64_t split = kInf;  // near/far split (uniform across the grid)
    int64_t qtot = 1;       // |Q_r| = near + far
    uint64_t theta_prev = 0;
    int warm = 0;
    int64_t r = 1;
    for (;;) {  // grid rounds, then small-frontier rounds while they apply, then grid rounds, ...
    bool go_small = false;
    for (;; r++) {
        RoundCnt* C = &ctrl->cnt[r % 3];
        const Sharded<int32_t> QC = queue_of(p, r);
        const Sharded<Desc> CL = chunks_of(p, r);
        // |Q_r| = |Q_{r-1}| + sum over CTAs of (inserts - extractions) in round r-1
        // warps 1 and 3, in parallel with warp 0's load_prefix: the previous round's |Q|
        // delta and min_Q delta (Delta* / Dijkstra)
        if (small_on(FUSE) && (threadIdx.x >> 5) == 2) {
            const int lane = lane_id();
            const int32_t* ce = p.cta_ext + ((r + 2) % 3) * kMaxCtas;
            int32_t se = 0;
            for (int i = lane; i < (int)gridDim.x; i += 32) se += __ldcg(ce + i);
            se = warp_sum(se);
            if (lane == 0) bc_ext = se;
        }
        if ((threadIdx.x >> 5) == 1 && r > 1) {
            const int lane = lane_id();
            const int64_t* cd = p.cta_delta + ((r + 2) % 3) * kMaxCtas;
            int64_t sdq = 0;
            for (int i = lane; i < (int)gridDim.x; i += 32) sdq += __ldcg((const long long*)(cd + i));
            sdq = warp_sum(sdq);
            if (lane == 0) bc_dq = sdq;
        }
        if (uses_min(POL) && FUSE && (threadIdx.x >> 5) == 3) {
            // (fusion kernels only: in the others this placement cost registers in the hot
            // loops, rmat24 Delta* +7 %; grid4096 / rgg4m Delta* gain 2 % from it)
            const int lane = lane_id();
            const uint64_t* cm = p.cta_min + ((r + 2) % 3) * kMaxCtas;
            uint64_t mn = kInf;
            for (int i = lane; i < (int)gridDim.x; i += 32) {
                const uint64_t x = __ldcg((const unsigned long long*)(cm + i));
                mn = x < mn ? x : mn;
            }
            mn = warp_min_u64(mn);
            if (lane == 0) bc_u[0] = mn;
        }
        W.set_round(queue_of(p, r + 1), C);  // (all warps are past the previous round's appends)
        load_prefix(QC, qpref);  // ends with __syncthreads
        if (r > 1 && !ls.resumed) qtot += bc_dq;
        int64_t qn = qpref[kSeg];  // near part of Q_r
        if (qtot == 0) break;      // while |Q| > 0
        if (r > p.max_rounds) {
            if (gtid == 0) ctrl->status = SSSP_ERR_ROUNDS;
            break;
        }
        // ---- small-frontier rounds: all of Q listed and at most kSmallQ ids -> CTA 0 runs the
        // rounds alone (every CTA takes the same decision from the same counters)
        const bool try_small = small_on(FUSE) && qtot == qn && qtot <= kSmallQ && bc_ext <= kSmallF && !ls.cool &&
                               !(p.flags & SSSP_RUN_NO_SMALL) && (r > 1 || ls.src_deg <= kSmallArcs);
        if (small_on(FUSE)) {
            __syncthreads();  // (every thread has read ls)
            if (threadIdx.x == 0) ls.resumed = ls.cool = 0;
        }
        if (try_small) {
            go_small = true;
            break;
        }
        uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0, tn = 0;
        int64_t dense = 0;
        if (STATS && gtid == 0) t0 = tn = globaltimer();
        if (gtid == 0) reset_cnt(&ctrl->cnt[(r + 1) % 3]);
        if (threadIdx.x == 0) tile_ctr[(r + 1) & 1] = tile_ctr[2 + ((r + 1) & 1)] = 0;  // last used in round r-1
        if (gtid < 2 * kSeg) {  // counters of slot (r+1)%3: written in round r+1, read in r+1 / r+2
            p.counters[((int64_t)(((r + 1) % 3) * 2) * kSeg + gtid) * kCntStride] = 0;
        }
        if (threadIdx.x == 0) {
            p.cta_delta[((r + 1) % 3) * kMaxCtas + blockIdx.x] = 0;
            p.cta_ext[((r + 1) % 3) * kMaxCtas + blockIdx.x] = 0;
        }

        // ---- ExtDist (Table tab:framework) and near/far maintenance
        uint64_t theta;
        // A round that lowers the split runs snapshot-style (Extract finishes before any
        // relax): a live relax could not tell a near id still listed from one Extract
        // just moved to the far part (DESIGN.md §5 near/far).
        bool snap = (p.flags & SSSP_RUN_SNAPSHOT) != 0;
        if (POL == SSSP_BELLMAN_FORD) {
            theta = kInf;
        } else if (POL == SSSP_DIJKSTRA || POL == SSSP_DELTA || POL == SSSP_DELTA_STEPPING) {
            // min_Q delta = min over the per-CTA minima of the previous round (fusion kernels:
            // warp 3 above, in parallel with load_prefix)
            if (!FUSE) {
                if (threadIdx.x < 32) {
                    const uint64_t* cm = p.cta_min + ((r + 2) % 3) * kMaxCtas;
                    uint64_t mn = kInf;
                    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
                        const uint64_t x = __ldcg((const unsigned long long*)(cm + i));
                        mn = x < mn ? x : mn;
                    }
                    mn = warp_min_u64(mn);
                    if (threadIdx.x == 0) bc_u[0] = mn;
                }
                __syncthreads();
            }
            const uint64_t minq = bc_u[0];  // <= min_{v in Q} delta[v] (exact in snapshot mode)
            if (POL == SSSP_DIJKSTRA) {
                theta = minq;
            } else if (POL == SSSP_DELTA_STEPPING && r > 1 && minq <= theta_prev) {
                theta = theta_prev;  // FinishCheck failed: Bellman-Ford substep on the same bucket (R19)
            } else {
                const uint64_t D = p.param;  // theta_i = i*Delta, skipping empty steps (reading R2)
                const uint64_t x = theta_prev > kInf - D ? kInf : theta_prev + D;
                const uint64_t y = (minq / D + (minq % D != 0)) * D;
                theta = x > y ? x : y;
                theta_prev = theta;
            }
        } else {  // rho
            uint64_t rho = p.param;
            if (!(p.flags & SSSP_RUN_NO_WARMUP) && (uint64_t)qtot > rho && warm < 2) {
                warm++;
                rho = rho / 10 ? rho / 10 : 1;  // reading R7
            }
            const uint64_t want = rho > kInf / (4 * kNearK) ? kInf / 4 : (uint64_t)kNearK * rho;
            // pull far keys in until the near part holds the rho smallest of Q (or all of Q)
            for (int it = 0; nearfar && qtot > qn && ((uint64_t)qtot <= rho || (uint64_t)qn < rho); it++) {
                uint64_t hi = kInf;
                if ((uint64_t)qtot > rho && it < 3) {
                    if (blockIdx.x == 0) {
                        const uint64_t tgt = want > kInf >> 4 ? want : want << it;
                        int64_t need = tgt >= (uint64_t)qtot ? qtot : (int64_t)tgt - qn;
                        need = need < 1 ? 1 : need;
                        const uint64_t h = need >= qtot - qn ? kInf
                                                             : far_quantile(p, split, qtot - qn, need, r * 4 + it,
                                                                            s_keys, sm, &bc_cnt);
                        if (threadIdx.x == 0) C->split = h;
                    }
                    grid_sync();
                    if (threadIdx.x == 0) bc_u[2] = __ldcg((const unsigned long long*)&C->split);
                    __syncthreads();
                    hi = bc_u[2];
                }
                far_to_near(p, QC, split, hi, W);
                dense += p.n;
                grid_sync();
                load_prefix(QC, qpref);
                qn = qpref[kSeg];
                split = hi;
            }
            const QueueVal qv{QC, qpref, p.dist};
            if (nearfar && (uint64_t)qn > 4 * want && qn > (int64_t)(p.n >> 5)) {
                // the near part grew far beyond the target: lower the split to about the
                // want-th smallest near key (CTA 0 + broadcast keeps it grid-uniform);
                // Extract then leaves the near ids above it to the far part
                if (blockIdx.x == 0) {
                    uint64_t s2 = sample_count((uint64_t)qn, want);
                    s2 = s2 > (uint64_t)kSmemSamples ? (uint64_t)kSmemSamples : s2;
                    for (uint64_t j = threadIdx.x; j < s2; j += blockDim.x)
                        s_keys[j] = qv((int64_t)sample_index(p.seed ^ 0x5EED5EEDull, r, j, (uint64_t)qn));
                    __syncthreads();
                    uint64_t k = (want * s2 + (uint64_t)qn - 1) / (uint64_t)qn;
                    k = k < 1 ? 1 : (k > s2 ? s2 : k);
                    const uint64_t h = cta_kth_smallest(SmemKey{s_keys}, (int64_t)s2, k, sm);
                    if (threadIdx.x == 0) C->split = h;
                }
                grid_sync();
                if (threadIdx.x == 0) bc_u[2] = __ldcg((const unsigned long long*)&C->split);
                __syncthreads();
                if (bc_u[2] < split) {
                    split = bc_u[2];
                    snap = true;
                }
            }
            if (STATS && gtid == 0) tn = globaltimer();
            const uint64_t s = sample_count((uint64_t)qn, rho);
            if ((uint64_t)qtot <= rho) {
                theta = kInf;  // |Q| <= rho: extract all
            } else if ((uint64_t)qn < rho) {
                theta = split;  // (near part short of rho after the pulls: extract all of it)
            } else if (!(p.flags & SSSP_RUN_RHO_EXACT) && s <= (uint64_t)kSmemSamples) {
                // every CTA draws the same samples of the near part (which holds the rho
                // smallest keys of Q) and selects the same theta: no barrier
                for (uint64_t j = threadIdx.x; j < s; j += blockDim.x)
                    s_keys[j] = qv((int64_t)sample_index(p.seed, r, j, (uint64_t)qn));
                __syncthreads();
                uint64_t k = (rho * s + (uint64_t)qn - 1) / (uint64_t)qn;
                k = k < 1 ? 1 : (k > s ? s : k);
                theta = s <= (uint64_t)kRankSelect ? cta_kth_by_rank(s_keys, (int)s, k, sm)
                                                   : cta_kth_smallest(SmemKey{s_keys}, (int64_t)s, k, sm);
            } else {
                if (blockIdx.x == 0) {
                    uint64_t th;
                    if (p.flags & SSSP_RUN_RHO_EXACT) {
                        th = cta_kth_smallest(qv, qn, rho, sm);
                    } else {
                        for (uint64_t j = threadIdx.x; j < s; j += blockDim.x)
                            p.samples[j] = qv((int64_t)sample_index(p.seed, r, j, (uint64_t)qn));
                        __syncthreads();
                        uint64_t k = (rho * s + (uint64_t)qn - 1) / (uint64_t)qn;
                        k = k < 1 ? 1 : (k > s ? s : k);
                        th = cta_kth_smallest(ArrayKey{p.samples}, (int64_t)s, k, sm);
                    }
                    if (threadIdx.x == 0) C->theta = th;
                }
                grid_sync();
                if (threadIdx.x == 0) bc_u[1] = __ldcg((const unsigned long long*)&C->theta);
                __syncthreads();
                theta = bc_u[1];
            }
        }
        W.split = split;
        // fusion in live rounds (FUSE kernels are launched for sparse graphs only, run.cu)
        W.fuse_theta = (FUSE && !snap) ? theta : 0;
        W.fbudget = p.fuse_budget;
        if (STATS && gtid == 0) t1 = globaltimer();

        // ---- phase A: Extract(theta) (+ light relax in live mode)
        uint64_t minrem = kInf;
        const uint64_t ta = STATS ? globaltimer() : 0;
#if SSSP_PROF
        for (int i = 0; i < kProf; i++) W.prof[i] = 0;  // phase-A only
#endif
        phase_a<POL, STATS, FUSE, BIDIR>(p, QC, qpref, CL, theta, snap, minrem, W, &tile_ctr[r & 1]);
        if (STATS && lane_id() == 0) {
            const unsigned long long ba = globaltimer() - ta;
            atomicAdd(&C->busy_a, ba);
            atomicMax(&C->busy_a_max, ba);
#if SSSP_PROF
            for (int i = 0; i < kProf; i++) atomicAdd(&C->prof[i], (unsigned long long)W.prof[i]);
#endif
#if SSSP_BAL  // balance probe: per-CTA sum and max of the warps' phase-A busy time
            atomicAdd(&bal[0], ba);
            atomicMax(&bal[1], ba);
#endif
        }
#if SSSP_BAL
        if (STATS) {
            __syncthreads();
            if (threadIdx.x == 0) {
                atomicMax(&C->prof[0], bal[0] / kWarps);  // max over CTAs of the CTA-mean busy
                atomicAdd(&C->prof[1], bal[0] / kWarps);  // sum over CTAs of the CTA-mean busy
                atomicAdd(&C->prof[2], bal[1]);           // sum over CTAs of the CTA-max busy
                bal[0] = bal[1] = 0;
            }
        }
#endif
#if SSSP_PROF
        for (int i = 0; i < kProf; i++) W.prof[i] = 0;
#endif
        flush_acc<POL, STATS, FUSE, BIDIR>(p, r, W);
        // this CTA's min over kept ids and successful WriteMins so far (Delta* / Dijkstra):
        // published before the barrier, so a round without phase-B work needs no second one
        auto publish_min = [&]() {
            uint64_t mn = warp_min_u64(minrem < W.acc.minsucc ? minrem : W.acc.minsucc);
            if (lane_id() == 0) red[threadIdx.x >> 5] = mn;
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int i = 1; i < kWarps; i++) mn = red[i] < mn ? red[i] : mn;
                p.cta_min[(r % 3) * kMaxCtas + blockIdx.x] = mn;
            }
        };
        if (uses_min(POL)) publish_min();
        grid_sync();
        if (STATS && gtid == 0) t2 = globaltimer();
        // ---- phase B: heavy chunks (+ light list in snapshot mode)
        bool phase_b_work;
        int32_t nl = 0;
        if (FUSE && !snap) {
            // fusion rounds rarely emit chunks: every warp sums the 33 chunk counters itself
            // (no CTA barrier), the prefix is built only if there is work (2.5 % on grid4096)
            const int lane = lane_id();
            int64_t c = CL.seg_count(lane);
            if (lane == 0) c += CL.seg_count(kShards);
            phase_b_work = warp_sum(c) > 0;  // (final after the grid barrier: the same in every warp)
            if (phase_b_work) load_prefix(CL, cpref);
        } else {
            if (threadIdx.x == 0) bc_nl = snap ? __ldcg(&C->nlight) : 0;  // (thread 0 is in warp 0: one barrier)
            load_prefix(CL, cpref);
            nl = bc_nl;
            phase_b_work = cpref[kSeg] + nl > 0;
        }
        if (phase_b_work) {
            const uint64_t tb = STATS ? globaltimer() : 0;
            // (the snapshot-style rounds with a light list keep the static order: handling the
            // light batches in the dynamic loop cost rmat24 rho 3 %, Delta* 6 %)
            phase_b<POL, STATS, FUSE, BIDIR>(p, CL, cpref, nl, W, warp_rank(), ((int64_t)gridDim.x * blockDim.x) >> 5,
                                             nl == 0 ? &tile_ctr[2 + (r & 1)] : nullptr);
            if (STATS && lane_id() == 0) atomicAdd(&C->busy_b, (unsigned long long)(globaltimer() - tb));
        }
        drain_pending<POL, STATS, FUSE, BIDIR>(p, W);  // deferred WriteMins count in min_Q
        if (uses_min(POL)) {
            if (phase_b_work) publish_min();  // now including phase B's WriteMins
            W.acc.minsucc = kInf;
        }
        if (phase_b_work) {
            flush_acc<POL, STATS, FUSE, BIDIR>(p, r, W);
            grid_sync();
        } else if (STATS) {
            grid_sync();
        }
        if (STATS && gtid == 0) t3 = globaltimer();

        if (STATS && gtid == 0) {
            const int64_t f = (int64_t)C->fsize;
            if (p.trace && r - 1 < p.trace_cap) {
                sssp_round* t = p.trace + (r - 1);
                t->qsize = qtot;
                t->fsize = f;
                t->edges = (int64_t)C->edges;
                t->inserts = (int64_t)C->inserts;
                t->succ = (int64_t)C->succ;
                t->theta = theta;
                t->nheavy = (int64_t)C->nheavy;
                t->t_theta_ns = (int64_t)(t1 - t0);
                t->t_extract_ns = (int64_t)(t2 - t1);
                t->t_relax_ns = (int64_t)(t3 - t2);
                t->qnear = qn;
                t->dense = dense;
                t->busy_a_ns = (int64_t)C->busy_a;
                t->busy_b_ns = (int64_t)C->busy_b;
                t->busy_a_max_ns = (int64_t)C->busy_a_max;
                t->fused = (int64_t)C->fused;
                t->t_near_ns = (int64_t)(tn - t0);
                for (int i = 0; i < kProf; i++) t->prof[i] = (int64_t)C->prof[i];
            }
            ctrl->tot_extracted += f;
            ctrl->tot_edges += (int64_t)C->edges;
            ctrl->tot_succ += (int64_t)C->succ;
            ctrl->tot_inserts += (int64_t)C->inserts;
            ctrl->tot_qscan += qn;
            ctrl->tot_dense += dense;
            ctrl->max_q = qtot > ctrl->max_q ? qtot : ctrl->max_q;
            ctrl->max_f = f > ctrl->max_f ? f : ctrl->max_f;
        }
    }
        if (!small_on(FUSE) || !go_small) break;
#if !SSSP_FUSE_UNIT
        if constexpr (small_on(FUSE)) {
        // ---- small-frontier rounds (outside the grid's round loop: no call or cold state
        // inside its register allocation)
        const Sharded<int32_t> QC = queue_of(p, r);
        const int32_t epoch = ls.epoch + 1;
        if (blockIdx.x == 0) {
            uint64_t minq = 0;
            if (uses_min(POL)) {
                if (threadIdx.x < 32) {
                    const uint64_t* cm = p.cta_min + ((r + 2) % 3) * kMaxCtas;
                    uint64_t mn = kInf;
                    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
                        const uint64_t x = __ldcg((const unsigned long long*)(cm + i));
                        mn = x < mn ? x : mn;
                    }
                    mn = warp_min_u64(mn);
                    if (threadIdx.x == 0) bc_u[0] = mn;
                }
                __syncthreads();
                minq = bc_u[0];
            }
            small_rounds<POL, STATS, FUSE, BIDIR>(p, r, qtot, theta_prev, warm, minq, QC, qpref, cpref, red);
            if (threadIdx.x == 0) {
                __threadfence();
                st_release_i32(&ctrl->sm_epoch, epoch);
                ls.epoch = epoch;
            }
        } else {
            if (threadIdx.x == 0)
                while (ld_acquire_i32(&ctrl->sm_epoch) < epoch) __nanosleep(128);
            if (threadIdx.x == 0) ls.epoch = epoch;
            __syncthreads();
        }
        const int64_t r_new = ld_volatile_i64(&ctrl->sm_r);
        const bool over = ld_volatile_i32(&ctrl->sm_end) != 0;
        qtot = ld_volatile_i64(&ctrl->sm_qtot);
        theta_prev = ld_volatile_u64(&ctrl->sm_theta_prev);
        warm = ld_volatile_i32(&ctrl->sm_warm);
        split = kInf;  // small rounds list all of Q
        if (threadIdx.x == 0) {
            tile_ctr[0] = tile_ctr[1] = tile_ctr[2] = tile_ctr[3] = 0;
            p.cta_delta[(r_new % 3) * kMaxCtas + blockIdx.x] = 0;
            p.cta_ext[(r_new % 3) * kMaxCtas + blockIdx.x] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            ls.cool = r_new == r;  // the first small round was too large: the grid runs it
            ls.resumed = 1;
        }
        r = r_new;
        if (over) break;
        }
#endif
    }
    if (gtid == 0) ctrl->rounds = r - 1;
    // S6 output: strip the flag bit (every reached vertex was extracted; INF stays INF)
    if (p.nofo) {  // compacted ids: out[v] = delta[nofo[v]] for every caller id v
        // A warp maps 512 consecutive ids per step: 4 coalesced 16-byte map loads per lane, then
        // 16 key loads in flight, then the stores (16-byte ones if the caller's array allows).
        // The pass is a chain of two dependent loads per step, so its length is steps per warp:
        // 7 on rmat24 (it was 28 with 4 ids per thread per step).  nofo is a 256-byte-aligned
        // workspace array.
        const auto strip = [](uint64_t x) { return (x != kInf && (x & kTop)) ? (x & kVal) : x; };
        const int64_t nblk = p.n_out / 512;
        const bool al16 = ((uintptr_t)p.out & 15) == 0;
        for (int64_t blk = gtid >> 5; blk < nblk; blk += gsize >> 5) {
            const int64_t v0 = blk * 512 + lane_id() * 4;
            int4 u4[4];
#pragma unroll
            for (int k = 0; k < 4; k++) u4[k] = __ldcg((const int4*)(p.nofo + v0 + k * 128));
            uint64_t x[16];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int32_t u[4] = {u4[k].x, u4[k].y, u4[k].z, u4[k].w};
#pragma unroll
                for (int j = 0; j < 4; j++)
                    x[k * 4 + j] = (u[j] < p.n || u[j] == src) ? __ldcg((const unsigned long long*)(p.dist + u[j])) : kInf;
            }
#pragma unroll
            for (int k = 0; k < 4; k++) {
                uint64_t* o = p.out + v0 + k * 128;
                if (al16) {
                    *(ulonglong2*)o = make_ulonglong2(strip(x[k * 4]), strip(x[k * 4 + 1]));
                    *(ulonglong2*)(o + 2) = make_ulonglong2(strip(x[k * 4 + 2]), strip(x[k * 4 + 3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++) o[j] = strip(x[k * 4 + j]);
                }
            }
        }
        for (int64_t v = nblk * 512 + gtid; v < p.n_out; v += gsize) {
            const int32_t u = p.nofo[v];
            const uint64_t x = (u < p.n || u == src) ? __ldcg((const unsigned long long*)(p.dist + u)) : kInf;
            p.out[v] = strip(x);
        }
    } else {
        for (int64_t i = gtid; i < p.n; i += gsize) {
            const uint64_t x = __ldcg((const unsigned long long*)(p.dist + i));
            if (x != kInf && (x & kTop)) p.dist[i] = x & kVal;
        }
    }
}

typedef void (*KernelFn)(RunParams);

// this translation unit's dynamic shared memory per CTA (its constants may be unit-specific)
static constexpr size_t smem_bytes(bool fuse) { return kSmemBase + (fuse ? kWarps * sizeof(FuseStage) : 0); }

// One object file (inst.cu) per (policy, bidirectional, fusion): the plain and the stats
// kernel and the shared memory they need.
struct KernelUnit {
    KernelFn plain, stats;
    size_t smem;
    int block;  // threads per CTA of this unit's kernels (SSSP_BLOCK may be unit-specific, build.py)
};
#define SSSP_DECLARE_UNIT(P, B, F) KernelUnit kernel_unit_##P##_##B##_##F();
#define SSSP_DECLARE_UNITS(P) \
    SSSP_DECLARE_UNIT(P, 0, 0) SSSP_DECLARE_UNIT(P, 0, 1) SSSP_DECLARE_UNIT(P, 1, 0) SSSP_DECLARE_UNIT(P, 1, 1)
SSSP_DECLARE_UNITS(0) SSSP_DECLARE_UNITS(1) SSSP_DECLARE_UNITS(2) SSSP_DECLARE_UNITS(3) SSSP_DECLARE_UNITS(4)
#undef SSSP_DECLARE_UNITS
#undef SSSP_DECLARE_UNIT

}  // namespace sssp
