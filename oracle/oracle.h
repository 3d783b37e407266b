/*
 * oracle.h — plain, slow, obviously-correct CPU reference for the stepping-SSSP
 * hot path of arXiv 2105.06145 (PAPER.md in /root/reference).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code, header, table or constant generator with the CUDA path
 * (paper_2105_06145_b200/, include/), and neither side includes the other.
 *
 * Citations: P:n = PAPER.md line n.
 *
 * Parity pins (tests/test_oracle.py, all -m "not gpu"):
 *   oracle_dijkstra        pinned by brute-force Bellman-Ford, scipy's Dijkstra,
 *                          closed forms (grid/chain/star/tree), golden examples.
 *   oracle_bellman_ford    pinned by closed forms and scipy (independent algorithms).
 *   oracle_certify         pinned by accepting exact distances and rejecting each
 *                          single-condition perturbation.
 *   oracle_stepping_sim    distances pinned to Dijkstra; rounds pinned by theorems
 *                          (BF = k_n+1, every policy >= k_n+1, Lemma num-ext,
 *                          Thm deltass, Thm rho-steps-un on tiny graphs).
 *   oracle_select_sampled  pinned by the statistical rank bound of App. cpam
 *                           and degenerate cases (|Q|<=rho, equal keys).
 */
#ifndef SSSP_ORACLE_H
#define SSSP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_INF UINT64_MAX

/* Textbook Dijkstra (Alg. 1 "Output: the graph distances",
 * P:224) with an indexed binary heap keyed by tentative distance.  If hops != NULL,
 * also returns, for every reached vertex, the fewest edges on a shortest path
 * (hop distance); k_n = max hops.  Returns number reached. */
int64_t oracle_dijkstra(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                        uint64_t *dist, int32_t *hops);

/* Same, but stops once `arc_budget` arcs have been scanned (bounded CPU
 * baseline sample).  Returns arcs scanned; *settled = vertices popped. */
int64_t oracle_dijkstra_budget(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                               uint64_t *dist, int64_t arc_budget, int64_t *settled);

/* Brute-force Bellman-Ford: up to n-1 synchronous passes over all
 * arcs, stopping early when a pass changes nothing.  Returns passes made. */
int64_t oracle_bellman_ford(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                            uint64_t *dist);

/* Breadth-first reachability/levels (unit-weight distances). level=-1 if unreached. */
int64_t oracle_bfs(int32_t n, const int32_t *off, const int32_t *idx, int32_t s, int32_t *level);

/* Optimality certificate for candidate distances d (w >= 1):
 *  (i) d[s]=0; (ii) every arc (u,v,w) with d[u]<INF has d[v] <= d[u]+w;
 *  (iii) every v != s with d[v]<INF has an in-arc (u,v,w) with d[u]+w = d[v];
 *  (iv) d[v]=INF iff v is unreachable.
 * Returns 0 if all hold, else the number (1..4) of the first failed condition;
 * *bad = offending vertex. */
int oracle_certify(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                   const uint64_t *d, int64_t *bad);

/* Policies of Table tab:framework. */
enum { ORACLE_RHO = 0, ORACLE_DELTA = 1, ORACLE_BF = 2, ORACLE_DIJKSTRA = 3, ORACLE_DELTA_STEPPING = 4 };
/* flags */
enum { ORACLE_RHO_EXACT = 1, ORACLE_RHO_WARMUP = 2 };

/* One row per round of the simulated Alg. 1. */
typedef struct {
    int64_t qsize;   /* |Q_r| before Extract                              */
    int64_t fsize;   /* |F_r| = vertices extracted                        */
    int64_t edges;   /* arcs scanned = sum of out-degrees of F_r          */
    int64_t inserts; /* vertices added to Q (not in Q after Extract)      */
    int64_t succ;    /* successful WriteMins (order dependent; info only) */
    uint64_t theta;  /* ExtDist value                                    */
    int64_t pad0, pad1;
} oracle_round;

/* Sequential simulation of Alg. 1 with snapshot semantics: F_r is
 * extracted with its keys, then every u in F_r relaxes N(u) with the key it had
 * at Extract (reading R8).  ExtDist per policy:
 *   BF:        theta = +inf
 *   DELTA:     theta_r = max(theta_{r-1}+D, ceil(min_Q/D)*D)  (reading R2)
 *   RHO:       theta = rho-th smallest key in Q (exact, flag)
 *              or the sampled estimate of oracle_select_sampled;
 *              |Q| <= rho -> +inf; warm-up rho/10 in the first two
 *              rounds with |Q| > rho (reading R7).
 *   DIJKSTRA:  theta = min_Q key
 *   DELTA_STEPPING: theta_i = i*Delta with FinishCheck: the same theta again while
 *              min_Q <= theta (substeps), else as DELTA        (reading R19)
 * Writes distances, per-round trace (up to trace_cap rows), and optional
 * per-vertex extraction counts.  Returns rounds, or -1 if max_rounds exceeded. */
int64_t oracle_stepping_sim(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                            int policy, uint64_t param, uint32_t flags, uint64_t seed, int64_t max_rounds,
                            uint64_t *dist, oracle_round *trace, int64_t trace_cap, int32_t *ext_count);

/* ExtDist of rho-stepping by sampling (App. cpam),
 * over the queue's keys in queue order keys[0..q):
 *   q <= rho          -> +inf (drain, reading R4)
 *   s = ceil(10*q/rho) + 10*(1 + floor(log2(q+1)))   (c = 10; reading R5)
 *   s = min(s, 65536)
 *   sample j in [0,s): index = splitmix64(seed ^ splitmix64((round<<32) | j)) mod q
 *   sort samples; k = clamp(ceil(rho*s/q), 1, s); theta = k-th smallest (1-based). */
uint64_t oracle_select_sampled(const uint64_t *keys, int64_t q, uint64_t rho, uint64_t seed, uint64_t round);

/* Exact rho-th smallest (1-based) of keys[0..q), or +inf when q <= rho. */
uint64_t oracle_select_exact(const uint64_t *keys, int64_t q, uint64_t rho);

#ifdef __cplusplus
}
#endif
#endif
