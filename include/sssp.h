/*
 * sssp.h — C ABI of the B200-native stepping-SSSP library (libsssp.so).
 *
 * Implements the data-parallel hot path of arXiv 2105.06145 "Efficient Stepping
 * Algorithms and Implementations for Parallel Shortest Paths" (/root/reference/
 * PAPER.md; P:n = PAPER.md line n):
 *   - the stepping algorithm framework, Alg. 1 (P:219-241 = P:756-777): per round
 *     theta = ExtDist(); F = Q.Extract(theta); for u in F, v in N(u):
 *     if WriteMin(delta[v], delta[u] + w(u,v)) then Q.Update(v);
 *   - its policies (Table tab:framework): rho-stepping, Delta*-stepping,
 *     Bellman-Ford, and Dijkstra's theta = min_Q;
 *   - the lazy-batched priority queue LaB-PQ (Table tab:interface
 *     P:196-211), array-based, held on the device as a flag bitmap
 *     plus a compacted queue.
 *
 * Conventions
 *   - Graphs are CSR: int32 offsets[n+1], int32 indices[m], uint32 weights[m]
 *     (weights >= 1).  Arcs are directed; an undirected graph stores both.
 *   - Distances are uint64; unreachable = SSSP_INF = 2^64-1.  All arithmetic is
 *     integer, so every policy returns bit-identical exact distances (Alg. 1
 *     "Output: the graph distances d(.)").
 *   - "d_" pointers are CUDA device pointers, "h_" pointers host pointers.  The
 *     library never allocates device memory: the caller passes a workspace of
 *     the size the *_workspace_bytes() query returns, and keeps every borrowed
 *     buffer alive until the matching *_destroy().
 *   - A stream is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work of a handle is ordered on that stream.  Handles are not
 *     thread-safe; use one handle per stream.
 *   - Every call returns an sssp_status; on error, sssp_last_error() returns a
 *     thread-local detail string.  No C++ exception crosses this boundary.
 */
#ifndef SSSP_H
#define SSSP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSSP_INF UINT64_MAX
#define SSSP_ABI_VERSION 1

typedef enum {
    SSSP_OK = 0,
    SSSP_ERR_INVALID = -1,       /* bad argument (null pointer, size, param, workspace too small)   */
    SSSP_ERR_INVALID_GRAPH = -2, /* SSSP_VALIDATE found a malformed CSR or a weight < 1             */
    SSSP_ERR_RANGE = -3,         /* vertex id outside [0, n)                                         */
    SSSP_ERR_CAPACITY = -4,      /* output buffer too small; the queue is left unchanged             */
    SSSP_ERR_CUDA = -5,          /* a CUDA runtime call or kernel failed                              */
    SSSP_ERR_ROUNDS = -6,        /* max_rounds exceeded (distances are then NOT final)                */
    SSSP_ERR_DEVICE = -7,        /* no usable sm_100 device / cooperative launch unsupported          */
    SSSP_ERR_INTERNAL = -8       /* a device-side capacity guard fired (a bug; distances not final)   */
} sssp_status;

/* ExtDist rules of Table tab:framework.  FinishCheck is empty for all. */
typedef enum {
    SSSP_RHO = 0,          /* theta = rho-th smallest key in Q; param = rho >= 1   */
    SSSP_DELTA = 1,        /* Delta*: theta_i = i*Delta, no FinishCheck;
                              param = Delta >= 1; empty steps skipped (reading R2)        */
    SSSP_BELLMAN_FORD = 2, /* theta = +inf; param ignored                            */
    SSSP_DIJKSTRA = 3,     /* theta = min_{v in Q} delta[v]; param ignored        */
    SSSP_DELTA_STEPPING = 4 /* theta_i = i*Delta WITH FinishCheck: the bucket is extracted again while
                              Q holds a key <= i*Delta (reading R19);
                              param = Delta >= 1                                                    */
} sssp_policy;

typedef void *sssp_stream_t; /* a cudaStream_t */

/* ---------------------------------------------------------------- SSSP handle */

typedef struct sssp_handle sssp_handle;

/* sssp_create flags */
#define SSSP_VALIDATE 1u /* check the CSR on the device at create time (one extra kernel) */
#define SSSP_NO_RELABEL 2u /* keep the caller's vertex ids inside the handle.  By default a
                            * power-law graph (m >= 20 n) with >= n/16 isolated vertices is
                            * renumbered inside the handle: the non-isolated vertices become
                            * 0..nz-1 (original order), so the run's distance array holds
                            * only them; runs map the source in and the distances back, the
                            * API is unchanged (workspace +20n bytes when m >= 20 n) */

/* Bytes of device workspace a handle for an n-vertex, m-arc graph needs (flags as
 * for sssp_create).  Holds an interleaved copy of the arcs ({head, weight}, 8m
 * bytes), the LaB-PQ (two queues; the in-Q flag is bit 63 of each distance
 * word), the heavy-vertex chunk map, theta samples, an internal distance array
 * and the control block.  Returns 0 if n or m is out of range. */
size_t sssp_workspace_bytes(int32_t n, int64_t m, uint32_t flags);

/* Create a handle over a device-resident CSR.
 *   n in [1, 2^31-2], m in [0, 2^31-1]; d_offsets[n+1], d_indices[m], d_weights[m]
 *   are BORROWED device arrays (never freed by the library).  d_offsets is read by
 *   every run; d_indices / d_weights only by the copy into the workspace that
 *   sssp_create enqueues on `stream` (they may be reused once that work is done,
 *   a later change to them is not seen by the handle).  d_workspace is a
 *   borrowed device buffer of ws_bytes >= sssp_workspace_bytes(n, m, flags),
 *   256-byte aligned.  stream orders all later work.
 * Errors: SSSP_ERR_INVALID (null/size/alignment), SSSP_ERR_INVALID_GRAPH (with
 * SSSP_VALIDATE: offsets[0] != 0, offsets[n] != m, offsets decreasing, an index
 * outside [0,n), or a weight < 1), SSSP_ERR_DEVICE, SSSP_ERR_CUDA. */
sssp_status sssp_create(int32_t n, int64_t m, const int32_t *d_offsets, const int32_t *d_indices,
                        const uint32_t *d_weights, void *d_workspace, size_t ws_bytes, sssp_stream_t stream,
                        uint32_t flags, sssp_handle **out);

/* sssp_run_opts.flags */
#define SSSP_RUN_RHO_EXACT 1u /* rho: exact rho-th smallest instead of sampling (test mode) */
#define SSSP_RUN_NO_WARMUP 2u /* rho: disable "10% of rho at the first two dense rounds" */
#define SSSP_RUN_STATS 4u     /* collect per-run counters (slower variant of the round loop)          */
#define SSSP_RUN_SNAPSHOT 8u  /* deterministic rounds: Extract completes before any relax of the round
                                 and every frontier vertex relaxes with its key at Extract (reading R8).
                                 Default ("live"): light vertices relax while Extract is still running,
                                 fewer barriers; distances are identical, round counts may differ.     */
#define SSSP_RUN_NO_FUSE 32u    /* live rounds on sparse graphs (m < 20 n): do not extract a vertex
                                   improved to <= theta on the spot (DESIGN.md fusion) */
#define SSSP_RUN_BIDIR 64u      /* UNDIRECTED graphs only (the caller guarantees every arc (u,v,w) has
                                   its reverse (v,u,w)): a light vertex first pulls
                                   delta[u] <- min_v delta[v] + w(v,u) over its arcs, then pushes
                                   (DESIGN.md bidirectional)                          */
#define SSSP_RUN_NO_NEARFAR 16u /* rho: list all of Q in the queue array every round instead of only
                                   its near part (keys <= split; DESIGN.md §5 near/far)              */
#define SSSP_RUN_NO_SMALL 128u  /* never hand rounds to one CTA: while |Q| <= 2048 (all listed) and a
                                   round's frontier has <= 32768 arcs, CTA 0 otherwise runs the rounds
                                   alone with CTA barriers (DESIGN.md §5 small rounds)  */

typedef struct {
    uint32_t flags;
    uint32_t fuse_budget;   /* fusion: vertices a warp may extract on the spot per round (0 = default:
                               96 for rho-stepping, 64 otherwise) */
    uint64_t seed;          /* rho sampling: counter-based generator seed (reading R6)      */
    int64_t max_rounds;     /* 0 = default (4n + 64); exceeded -> SSSP_ERR_ROUNDS                     */
    void *d_trace;          /* nullable device sssp_round[trace_cap]; filled when SSSP_RUN_STATS      */
    int64_t trace_cap;
    int32_t *d_ext_count;   /* nullable device int32[n]: extractions per vertex (Lemma num-ext) */
    uint32_t fuse_depth;    /* fusion: hops a local search may go from its extracted seed (0 = default:
                               10 for rho-stepping, unbounded for Delta*-stepping) */
    uint32_t reserved;      /* must be 0 */
} sssp_run_opts;

/* One row per round (Alg. 1 iteration of the while loop). */
typedef struct {
    int64_t qsize;   /* |Q_r| before Extract                                   */
    int64_t fsize;   /* |F_r| extracted                                         */
    int64_t edges;   /* arcs scanned = sum of out-degrees over F_r              */
    int64_t inserts; /* ids added to Q this round (were not in Q after Extract) */
    int64_t succ;    /* successful WriteMins (schedule dependent)               */
    uint64_t theta;  /* ExtDist value                                          */
    int64_t nheavy;  /* extracted vertices relaxed through the heavy-chunk path */
    int64_t t_theta_ns;   /* device time of ExtDist (globaltimer, CTA 0 view)          */
    int64_t t_extract_ns; /* device time of Extract (+ fused light relax)             */
    int64_t t_relax_ns;   /* device time of the remaining relax phase                 */
    int64_t qnear;        /* ids listed in the queue array (near part of Q) and scanned  */
    int64_t dense;        /* vertices read by near/far dense passes this round           */
    int64_t busy_a_ns;    /* sum over warps of time spent in phase A before its barrier  */
    int64_t busy_b_ns;    /* sum over warps of time spent in phase B before its barrier  */
    int64_t busy_a_max_ns; /* the slowest warp's phase-A time (busy_a_ns / warps = mean)  */
    int64_t fused;        /* vertices extracted by fusion this round (included in fsize) */
    int64_t t_near_ns;    /* part of t_theta_ns spent on near/far pulls and shrinks      */
    int64_t prof[8];      /* -DSSSP_PROF=1 builds only (else 0), phase A summed over warps:
                             SM cycles in scan / take (delete + CSR row) / light relax /
                             queue flush / fuse_drain, fuse_drain batches, relax steps,
                             SM cycles in relax steps (parts overlap: flush and relax
                             steps also count inside the relax and fuse parts)            */
    int64_t small;        /* 1: a small-frontier round, run by CTA 0 alone                */
} sssp_round;

typedef struct {
    int64_t rounds;         /* rounds executed                                   */
    int64_t extracted;      /* sum |F_r|          (STATS only)                  */
    int64_t edges;          /* sum E_r            (STATS only)                  */
    int64_t succ;           /* sum successful WriteMin (STATS only)             */
    int64_t inserts;        /* sum inserts        (STATS only)                  */
    int64_t queue_scanned;  /* sum |Q_r|          (STATS only)                  */
    int64_t max_queue;      /* max |Q_r|          (STATS only)                  */
    int64_t max_frontier;   /* max |F_r|          (STATS only)                  */
    int64_t dense_scanned;  /* sum of near/far dense-pass vertex reads (STATS)  */
    int32_t grid_blocks;    /* persistent-kernel CTAs                           */
    int32_t block_threads;  /* threads per CTA                                  */
    double kernel_ms;       /* device time of the round-loop launch (CUDA events on the handle's stream) */
} sssp_run_stats;

/* Single-source shortest paths from `source` with the given policy (Alg. 1).
 *   d_dist_out: caller-owned device uint64[n]; receives the exact distances
 *   (SSSP_INF if unreachable).  Also used as the live tentative-distance array
 *   delta during the run, unless the handle compacted isolated vertices (see
 *   SSSP_NO_RELABEL): then delta is in the workspace and the last pass of the run
 *   writes every entry of d_dist_out.  stats: nullable host struct.
 * The whole run is ONE persistent cooperative kernel launch on the handle's
 * stream; the call then synchronises the stream to report device-side status.
 * Errors: SSSP_ERR_RANGE (source outside [0,n)), SSSP_ERR_INVALID (param == 0 for
 * RHO/DELTA, null d_dist_out, unknown policy), SSSP_ERR_ROUNDS, SSSP_ERR_CUDA. */
sssp_status sssp_run(sssp_handle *h, int32_t source, sssp_policy policy, uint64_t param, uint64_t *d_dist_out,
                     sssp_run_stats *stats);

/* sssp_run with options (opts nullable = defaults). */
sssp_status sssp_run_ex(sssp_handle *h, int32_t source, sssp_policy policy, uint64_t param,
                        const sssp_run_opts *opts, uint64_t *d_dist_out, sssp_run_stats *stats);

/* End-to-end variant: runs into the workspace's internal distance array, then
 * copies the n distances to HOST memory h_dist_out (pinned memory recommended)
 * and synchronises.  Same errors as sssp_run. */
sssp_status sssp_run_host(sssp_handle *h, int32_t source, sssp_policy policy, uint64_t param, uint64_t *h_dist_out,
                          sssp_run_stats *stats);

/* Multi-source batch with read-back, the end-to-end call for many sources: runs
 * h_sources[0..k) one after another and copies each result to HOST memory
 * h_dist_out[i*n .. (i+1)*n) (pinned memory recommended).  The read-back of run i (a
 * second stream, two internal distance buffers) overlaps run i+1, so the batch costs
 * about max(kernel, copy) per source instead of their sum.  opts as for sssp_run_ex
 * except SSSP_RUN_STATS (per run only).  stats (nullable): rounds summed over the batch,
 * kernel_ms = the whole batch including read-backs.  Synchronous.  Errors as sssp_run,
 * plus SSSP_ERR_INVALID for k < 0, NULL buffers or SSSP_RUN_STATS. */
sssp_status sssp_run_batch_host(sssp_handle *h, const int32_t *h_sources, int32_t k, sssp_policy policy,
                                uint64_t param, const sssp_run_opts *opts, uint64_t *h_dist_out,
                                sssp_run_stats *stats);

/* Releases host-side state only; never frees caller memory. */
sssp_status sssp_destroy(sssp_handle *h);

/* ---------------------------------------------------------------- LaB-PQ */

/* A standalone device LaB-PQ over a universe of ids [0, n) whose keys are the
 * borrowed device array d_keys[n] (the mapping function delta; read at
 * Extract time, so key changes between Update and Extract are honoured). */
typedef struct sssp_pq sssp_pq;

size_t sssp_pq_workspace_bytes(int32_t n);

/* Errors: SSSP_ERR_INVALID (n out of [1, 2^31-2], null pointer, small workspace). */
sssp_status sssp_pq_create(int32_t n, const uint64_t *d_keys, void *d_workspace, size_t ws_bytes,
                           sssp_stream_t stream, sssp_pq **out);

/* Batch Update (Table tab:interface): for each id in d_ids[0..count),
 * insert it if absent, else merely notify (a no-op: keys are read lazily).
 * Duplicates within or across batches are allowed; each id is stored once.
 * Asynchronous, stream-ordered.  An id outside [0,n) is skipped and latches a
 * device error flag reported as SSSP_ERR_RANGE by the next synchronous call
 * (sssp_pq_size / _extract / _select / _reduce_min / _queue). */
sssp_status sssp_pq_update(sssp_pq *q, const int32_t *d_ids, int64_t count);

/* Extract(theta): writes every queued id with d_keys[id] <=
 * theta to d_out[0..*h_count) in unspecified order and deletes them from Q.
 * Exclusive with other calls (stream order).  Synchronous: *h_count is host
 * memory.  If more than cap ids qualify: SSSP_ERR_CAPACITY, *h_count = the
 * number that qualify, and Q is unchanged.  A range error latched by an earlier
 * update is reported by this call after the extract has run (*h_count valid).
 * One launch (two if cap < n: the qualifying ids are counted first) and one
 * synchronisation. */
sssp_status sssp_pq_extract(sssp_pq *q, uint64_t theta, int32_t *d_out, int64_t cap, int64_t *h_count);

/* |Q| (synchronous). */
sssp_status sssp_pq_size(sssp_pq *q, int64_t *h_size);

/* ExtDist of rho-stepping over the current Q (synchronous):
 *   mode SSSP_SELECT_SAMPLED: the paper's sampling estimate (P:301, P:1373-1376,
 *     App. cpam) with the counter-based generator of reading R6
 *     (round = 0);
 *   mode SSSP_SELECT_EXACT: the exact rho-th smallest key.
 * |Q| <= rho -> SSSP_INF (extract everything).  rho == 0 -> SSSP_ERR_INVALID. */
#define SSSP_SELECT_SAMPLED 0u
#define SSSP_SELECT_EXACT 1u
sssp_status sssp_pq_select(sssp_pq *q, uint64_t rho, uint64_t seed, uint32_t mode, uint64_t *h_theta);

/* Reduce with (min, keys): min_{id in Q} d_keys[id], SSSP_INF if empty. */
sssp_status sssp_pq_reduce_min(sssp_pq *q, uint64_t *h_min);

/* Copy the queue's ids in internal order to d_out (test hook: lets a checker
 * replay the sampled selector on the same order).  SSSP_ERR_CAPACITY if cap < |Q|. */
sssp_status sssp_pq_queue(sssp_pq *q, int32_t *d_out, int64_t cap, int64_t *h_count);

sssp_status sssp_pq_destroy(sssp_pq *q);

/* ---------------------------------------------------------------- errors / info */

const char *sssp_status_string(sssp_status s);
const char *sssp_last_error(void);
int32_t sssp_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SSSP_H */
