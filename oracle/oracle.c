/*
 * oracle.c — plain CPU reference for the stepping-SSSP hot path (see oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may call this.  No code is shared with the
 * CUDA path.  Everything here is sequential and written for readability.
 *
 * Build: gcc -O2 -fPIC -shared oracle.c -o liboracle.so
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Indexed binary min-heap over (key, vertex) with decrease-key.       */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t *heap; /* heap[i] = vertex      */
    int32_t *pos;  /* pos[v] = index or -1  */
    const uint64_t *key;
    int32_t size;
} iheap;

static int heap_less(const iheap *h, int32_t a, int32_t b) {
    uint64_t ka = h->key[a], kb = h->key[b];
    return ka < kb || (ka == kb && a < b);
}
static void heap_swap(iheap *h, int32_t i, int32_t j) {
    int32_t a = h->heap[i], b = h->heap[j];
    h->heap[i] = b;
    h->heap[j] = a;
    h->pos[b] = i;
    h->pos[a] = j;
}
static void sift_up(iheap *h, int32_t i) {
    while (i > 0) {
        int32_t p = (i - 1) / 2;
        if (!heap_less(h, h->heap[i], h->heap[p])) break;
        heap_swap(h, i, p);
        i = p;
    }
}
static void sift_down(iheap *h, int32_t i) {
    for (;;) {
        int32_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->size && heap_less(h, h->heap[l], h->heap[m])) m = l;
        if (r < h->size && heap_less(h, h->heap[r], h->heap[m])) m = r;
        if (m == i) break;
        heap_swap(h, i, m);
        i = m;
    }
}
/* insert v, or restore order after key[v] decreased */
static void heap_push_or_decrease(iheap *h, int32_t v) {
    if (h->pos[v] < 0) {
        h->heap[h->size] = v;
        h->pos[v] = h->size;
        h->size++;
    }
    sift_up(h, h->pos[v]);
}
static int32_t heap_pop(iheap *h) {
    int32_t v = h->heap[0];
    h->size--;
    if (h->size > 0) {
        h->heap[0] = h->heap[h->size];
        h->pos[h->heap[0]] = 0;
        sift_down(h, 0);
    }
    h->pos[v] = -1;
    return v;
}

static int64_t dijkstra_impl(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                             uint64_t *dist, int32_t *hops, int64_t arc_budget, int64_t *settled_out) {
    iheap h;
    h.heap = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    h.pos = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    h.key = dist;
    h.size = 0;
    for (int32_t v = 0; v < n; v++) {
        dist[v] = ORACLE_INF;
        h.pos[v] = -1;
        if (hops) hops[v] = -1;
    }
    /* 1. dist[.] = INF; dist[s] = 0; push s */
    dist[s] = 0;
    if (hops) hops[s] = 0;
    heap_push_or_decrease(&h, s);
    int64_t reached = 0, scanned = 0, settled = 0;
    while (h.size > 0) {
        if (arc_budget >= 0 && scanned >= arc_budget) break;
        /* 2. pop the minimum u; relax every arc (u, v, w) */
        int32_t u = heap_pop(&h);
        settled++;
        uint64_t du = dist[u]; /* finite: only reached vertices enter the heap */
        for (int64_t e = off[u]; e < off[u + 1]; e++) {
            int32_t v = idx[e];
            uint64_t c = du + (uint64_t)w[e];
            scanned++;
            if (c < dist[v]) {
                dist[v] = c;
                if (hops) hops[v] = hops[u] + 1;
                heap_push_or_decrease(&h, v);
            } else if (hops && c == dist[v] && hops[u] + 1 < hops[v]) {
                /* equal length, fewer edges (hop distance P:714-716).  u has
                 * dist[u] < dist[v] (w >= 1), so v is not yet popped. */
                hops[v] = hops[u] + 1;
            }
        }
    }
    for (int32_t v = 0; v < n; v++) reached += dist[v] != ORACLE_INF;
    free(h.heap);
    free(h.pos);
    if (settled_out) *settled_out = settled;
    return arc_budget >= 0 ? scanned : reached;
}

int64_t oracle_dijkstra(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                        uint64_t *dist, int32_t *hops) {
    return dijkstra_impl(n, off, idx, w, s, dist, hops, -1, NULL);
}

int64_t oracle_dijkstra_budget(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                               uint64_t *dist, int64_t arc_budget, int64_t *settled) {
    return dijkstra_impl(n, off, idx, w, s, dist, NULL, arc_budget < 0 ? 0 : arc_budget, settled);
}

/* ------------------------------------------------------------------ */
/* Brute-force Bellman-Ford: synchronous passes over every arc.         */
/* ------------------------------------------------------------------ */
int64_t oracle_bellman_ford(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                            uint64_t *dist) {
    uint64_t *prev = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    for (int32_t v = 0; v < n; v++) dist[v] = ORACLE_INF;
    dist[s] = 0;
    int64_t passes = 0;
    for (int64_t it = 0; it < (int64_t)n - 1 || it == 0; it++) {
        memcpy(prev, dist, (size_t)n * sizeof(uint64_t));
        int changed = 0;
        for (int32_t u = 0; u < n; u++) {
            if (prev[u] == ORACLE_INF) continue;
            for (int64_t e = off[u]; e < off[u + 1]; e++) {
                uint64_t c = prev[u] + (uint64_t)w[e];
                if (c < dist[idx[e]]) {
                    dist[idx[e]] = c;
                    changed = 1;
                }
            }
        }
        passes++;
        if (!changed) break;
    }
    free(prev);
    return passes;
}

/* ------------------------------------------------------------------ */
/* BFS levels.                                                         */
/* ------------------------------------------------------------------ */
int64_t oracle_bfs(int32_t n, const int32_t *off, const int32_t *idx, int32_t s, int32_t *level) {
    int32_t *q = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    for (int32_t v = 0; v < n; v++) level[v] = -1;
    int64_t head = 0, tail = 0;
    level[s] = 0;
    q[tail++] = s;
    while (head < tail) {
        int32_t u = q[head++];
        for (int64_t e = off[u]; e < off[u + 1]; e++) {
            int32_t v = idx[e];
            if (level[v] < 0) {
                level[v] = level[u] + 1;
                q[tail++] = v;
            }
        }
    }
    free(q);
    return tail;
}

/* ------------------------------------------------------------------ */
/* Optimality certificate.                                             */
/* ------------------------------------------------------------------ */
int oracle_certify(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                   const uint64_t *d, int64_t *bad) {
    *bad = -1;
    if (d[s] != 0) { *bad = s; return 1; }
    /* (ii) no arc can improve d; also mark vertices having a tight in-arc */
    char *tight = (char *)calloc((size_t)n, 1);
    for (int32_t u = 0; u < n; u++) {
        if (d[u] == ORACLE_INF) continue;
        for (int64_t e = off[u]; e < off[u + 1]; e++) {
            int32_t v = idx[e];
            uint64_t c = d[u] + (uint64_t)w[e];
            if (d[v] > c) { *bad = v; free(tight); return 2; }
            if (d[v] == c) tight[v] = 1;
        }
    }
    /* (iii) every finite d[v], v != s, is achieved by a tight arc */
    for (int32_t v = 0; v < n; v++) {
        if (v != s && d[v] != ORACLE_INF && !tight[v]) { *bad = v; free(tight); return 3; }
    }
    free(tight);
    /* (iv) INF exactly on unreachable vertices */
    int32_t *lvl = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    oracle_bfs(n, off, idx, s, lvl);
    for (int32_t v = 0; v < n; v++) {
        if ((lvl[v] < 0) != (d[v] == ORACLE_INF)) { *bad = v; free(lvl); return 4; }
    }
    free(lvl);
    return 0;
}

/* ------------------------------------------------------------------ */
/* rho-th element selection (App. cpam).                   */
/* ------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

uint64_t oracle_select_sampled(const uint64_t *keys, int64_t q, uint64_t rho, uint64_t seed, uint64_t round) {
    if (q <= 0 || (uint64_t)q <= rho) return ORACLE_INF; /* partial extract: drain */
    /* s = c(|Q|/rho + log|Q|), c = 10, log x := 1 + floor(log2(x+1)) */
    uint64_t lg = 0;
    for (uint64_t x = (uint64_t)q + 1; x > 1; x >>= 1) lg++;
    uint64_t s = (10 * (uint64_t)q + rho - 1) / rho + 10 * (1 + lg);
    if (s > 65536) s = 65536;
    uint64_t *smp = (uint64_t *)malloc(s * sizeof(uint64_t));
    for (uint64_t j = 0; j < s; j++) {
        uint64_t r = splitmix64(seed ^ splitmix64((round << 32) | j));
        smp[j] = keys[r % (uint64_t)q];
    }
    qsort(smp, s, sizeof(uint64_t), cmp_u64); /* "sort the samples" */
    uint64_t k = (rho * s + (uint64_t)q - 1) / (uint64_t)q; /* the (rho*s/n)-th one */
    if (k < 1) k = 1;
    if (k > s) k = s;
    uint64_t th = smp[k - 1];
    free(smp);
    return th;
}

uint64_t oracle_select_exact(const uint64_t *keys, int64_t q, uint64_t rho) {
    if (q <= 0 || (uint64_t)q <= rho) return ORACLE_INF;
    uint64_t *c = (uint64_t *)malloc((size_t)q * sizeof(uint64_t));
    memcpy(c, keys, (size_t)q * sizeof(uint64_t));
    qsort(c, (size_t)q, sizeof(uint64_t), cmp_u64);
    uint64_t th = c[rho - 1];
    free(c);
    return th;
}

/* ------------------------------------------------------------------ */
/* Alg. 1, the stepping framework, simulated sequentially.              */
/* ------------------------------------------------------------------ */
static uint64_t sat_add(uint64_t a, uint64_t b) { return a > ORACLE_INF - b ? ORACLE_INF : a + b; }

int64_t oracle_stepping_sim(int32_t n, const int32_t *off, const int32_t *idx, const uint32_t *w, int32_t s,
                            int policy, uint64_t param, uint32_t flags, uint64_t seed, int64_t max_rounds,
                            uint64_t *dist, oracle_round *trace, int64_t trace_cap, int32_t *ext_count) {
    char *inQ = (char *)calloc((size_t)n, 1);
    int32_t *Q = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *Qn = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *F = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    uint64_t *Fd = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    uint64_t *keys = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    if (ext_count) memset(ext_count, 0, (size_t)n * sizeof(int32_t));

    /* line 1-2: delta[.] = +inf; delta[s] = 0; Q.Update(s) */
    for (int32_t v = 0; v < n; v++) dist[v] = ORACLE_INF;
    dist[s] = 0;
    int64_t q = 0;
    Q[q++] = s;
    inQ[s] = 1;

    uint64_t theta_prev = 0;
    int64_t warm_rounds = 0;
    int64_t round = 0;
    while (q > 0) { /* line 3: while |Q| > 0 */
        if (round >= max_rounds) { round = -1; break; }
        round++;
        /* ExtDist (Table tab:framework) */
        uint64_t theta;
        uint64_t minq = ORACLE_INF;
        for (int64_t i = 0; i < q; i++) {
            keys[i] = dist[Q[i]];
            if (keys[i] < minq) minq = keys[i];
        }
        if (policy == ORACLE_BF) {
            theta = ORACLE_INF;
        } else if (policy == ORACLE_DIJKSTRA) {
            theta = minq;
        } else if (policy == ORACLE_DELTA) {
            uint64_t D = param;
            uint64_t a = sat_add(theta_prev, D);
            uint64_t b = (minq / D + (minq % D != 0)) * D; /* ceil(min_Q / D) * D; min_Q < 2^63 */
            theta = a > b ? a : b;
            theta_prev = theta;
        } else if (policy == ORACLE_DELTA_STEPPING) {
            /* Delta-stepping with FinishCheck (Table tab:framework P:791): theta = i*Delta,
             * and "if no new delta[v] < i*Delta, i <- i+1": while Q still holds a key <= i*Delta the
             * same bucket is extracted again (a Bellman-Ford substep, reading R19); otherwise i
             * advances, skipping empty buckets as for Delta* (reading R2). */
            uint64_t D = param;
            if (round > 1 && minq <= theta_prev) {
                theta = theta_prev;
            } else {
                uint64_t a = sat_add(theta_prev, D);
                uint64_t b = (minq / D + (minq % D != 0)) * D;
                theta = a > b ? a : b;
            }
            theta_prev = theta;
        } else { /* RHO */
            uint64_t rho = param;
            if ((flags & ORACLE_RHO_WARMUP) && (uint64_t)q > rho && warm_rounds < 2) {
                warm_rounds++;
                rho = rho / 10 ? rho / 10 : 1;
            }
            if (flags & ORACLE_RHO_EXACT)
                theta = oracle_select_exact(keys, q, rho);
            else
                theta = oracle_select_sampled(keys, q, rho, seed, (uint64_t)round);
        }
        /* line 4: F = Q.Extract(theta), with each key snapshotted */
        int64_t nf = 0, nq = 0, edges = 0;
        for (int64_t i = 0; i < q; i++) {
            int32_t v = Q[i];
            if (dist[v] <= theta) {
                F[nf] = v;
                Fd[nf] = dist[v];
                nf++;
                inQ[v] = 0;
                edges += off[v + 1] - off[v];
                if (ext_count) ext_count[v]++;
            } else {
                Qn[nq++] = v;
            }
        }
        /* lines 4-6: for u in F, v in N(u): if WriteMin(delta[v], delta[u]+w) then Q.Update(v) */
        int64_t inserts = 0, succ = 0;
        for (int64_t i = 0; i < nf; i++) {
            int32_t u = F[i];
            for (int64_t e = off[u]; e < off[u + 1]; e++) {
                int32_t v = idx[e];
                uint64_t c = Fd[i] + (uint64_t)w[e];
                if (c < dist[v]) {
                    dist[v] = c;
                    succ++;
                    if (!inQ[v]) {
                        inQ[v] = 1;
                        Qn[nq++] = v;
                        inserts++;
                    }
                }
            }
        }
        if (trace && round - 1 < trace_cap) {
            oracle_round *t = &trace[round - 1];
            t->qsize = q;
            t->fsize = nf;
            t->edges = edges;
            t->inserts = inserts;
            t->succ = succ;
            t->theta = theta;
            t->pad0 = t->pad1 = 0;
        }
        int32_t *tmp = Q;
        Q = Qn;
        Qn = tmp;
        q = nq;
        /* FinishCheck: none for BF, Delta*, rho, Dijkstra */
    }
    free(inQ);
    free(Q);
    free(Qn);
    free(F);
    free(Fd);
    free(keys);
    return round;
}
