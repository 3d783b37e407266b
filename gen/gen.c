/*
 * gen.c — seeded synthetic graph generators (CSR, int32 offsets/indices,
 * uint32 weights).  This module is INPUT PLUMBING shared by the oracle side and
 * the CUDA side; it holds none of the SSSP method's arithmetic (no relaxation,
 * no priority queue, no thresholds).
 *
 * Workload recipes (SURVEY.md §8(d) "Concrete synthetic
 * inputs"), standing in for the paper's graphs:
 *   - 2D 4-neighbour grid, one hashed weight per undirected edge.
 *   - R-MAT(a,b,c,d), ef*2^scale draws, symmetrised, self-loops dropped,
 *     deduplicated; weight per unordered pair from a hash.
 *   - random geometric kNN graph (k nearest, Euclidean, ties -> lower id),
 *     symmetrised by union, weight = llround(len*1e6)+1.
 *   - G(n, draws) random graph (directed or symmetrised) for tests.
 * Every random value is a counter-based splitmix64 hash of (seed, key), so the
 * output is bit-identical for any thread count and edge order.
 *
 * Build: gcc -O2 -fopenmp -fPIC -shared -ffp-contract=off gen.c -o libgen.so -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t n;
    int64_t m;
    int32_t *offsets; /* n+1 */
    int32_t *indices; /* m   */
    uint32_t *weights; /* m   */
    double *xy;        /* optional 2n coordinates (RGG), else NULL */
} gen_graph;

static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
static inline uint64_t hkey(uint64_t seed, uint64_t key) { return splitmix64(seed ^ splitmix64(key)); }
static inline double unit53(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

/* weight modes */
enum { W_UNIFORM = 0, W_LOGUNIFORM = 1, W_CONST = 2 };

static inline uint32_t pair_weight(uint64_t wseed, int mode, uint32_t wparam, uint32_t a, uint32_t b) {
    uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
    uint64_t h = hkey(wseed, ((uint64_t)lo << 32) | hi);
    if (mode == W_UNIFORM) return 1u + (uint32_t)(h % (uint64_t)wparam); /* [1, wparam] */
    if (mode == W_LOGUNIFORM) {                                            /* floor(2^(L u)) in [1, 2^L-1] */
        double u = unit53(h);
        double w = floor(exp2((double)wparam * u));
        double wmax = ldexp(1.0, (int)wparam) - 1.0;
        if (w < 1.0) w = 1.0;
        if (w > wmax) w = wmax;
        return (uint32_t)w;
    }
    return wparam; /* W_CONST */
}

void gen_free(gen_graph *g) {
    if (!g) return;
    free(g->offsets);
    free(g->indices);
    free(g->weights);
    free(g->xy);
    free(g);
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
static void sort_row(int32_t *p, int64_t len) {
    if (len < 24) {
        for (int64_t i = 1; i < len; i++) {
            int32_t v = p[i];
            int64_t j = i - 1;
            while (j >= 0 && p[j] > v) { p[j + 1] = p[j]; j--; }
            p[j + 1] = v;
        }
    } else {
        qsort(p, (size_t)len, sizeof(int32_t), cmp_i32);
    }
}

/*
 * Build a CSR from `cnt` arcs given as (src[i], dst[i]) pairs; if symmetrise,
 * each pair also contributes (dst, src).  Self-loops are dropped when
 * drop_self; duplicate arcs are always removed; rows end up sorted by target.
 * Weights: per unordered pair hash (symmetric), see pair_weight.
 */
static gen_graph *csr_from_pairs(int32_t n, int64_t cnt, const uint32_t *src, const uint32_t *dst, int symmetrise,
                                 int drop_self, uint64_t wseed, int wmode, uint32_t wparam) {
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!deg) return NULL;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; i++) {
        uint32_t u = src[i], v = dst[i];
        if (drop_self && u == v) continue;
        __atomic_fetch_add(&deg[u], 1, __ATOMIC_RELAXED);
        if (symmetrise) __atomic_fetch_add(&deg[v], 1, __ATOMIC_RELAXED);
    }
    int64_t *start = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    int64_t acc = 0;
    for (int32_t v = 0; v < n; v++) { start[v] = acc; acc += deg[v]; }
    start[n] = acc;
    int64_t raw = acc;
    int32_t *tmp = (int32_t *)malloc((size_t)(raw ? raw : 1) * sizeof(int32_t));
    int64_t *cur = deg; /* reuse as cursor */
    memcpy(cur, start, ((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < cnt; i++) {
        uint32_t u = src[i], v = dst[i];
        if (drop_self && u == v) continue;
        int64_t p = __atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED);
        tmp[p] = (int32_t)v;
        if (symmetrise) {
            int64_t q = __atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED);
            tmp[q] = (int32_t)u;
        }
    }
    /* sort each row, count unique */
    int64_t *uniq = cur;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int32_t v = 0; v < n; v++) {
        int64_t b = start[v], e = start[v + 1];
        sort_row(tmp + b, e - b);
        int64_t k = 0;
        for (int64_t i = b; i < e; i++)
            if (i == b || tmp[i] != tmp[i - 1]) k++;
        uniq[v] = k;
    }
    gen_graph *g = (gen_graph *)calloc(1, sizeof(gen_graph));
    g->n = n;
    g->offsets = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    acc = 0;
    int64_t *nstart = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    for (int32_t v = 0; v < n; v++) { nstart[v] = acc; g->offsets[v] = (int32_t)acc; acc += uniq[v]; }
    nstart[n] = acc;
    g->offsets[n] = (int32_t)acc;
    g->m = acc;
    g->indices = (int32_t *)malloc((size_t)(acc ? acc : 1) * sizeof(int32_t));
    g->weights = (uint32_t *)malloc((size_t)(acc ? acc : 1) * sizeof(uint32_t));
#pragma omp parallel for schedule(dynamic, 1024)
    for (int32_t v = 0; v < n; v++) {
        int64_t b = start[v], e = start[v + 1], o = nstart[v];
        for (int64_t i = b; i < e; i++) {
            if (i == b || tmp[i] != tmp[i - 1]) {
                g->indices[o] = tmp[i];
                g->weights[o] = pair_weight(wseed, wmode, wparam, (uint32_t)v, (uint32_t)tmp[i]);
                o++;
            }
        }
    }
    free(tmp);
    free(start);
    free(nstart);
    free(deg);
    return g;
}

/* 2D 4-neighbour grid, id = r*cols + c, weight per undirected edge. */
gen_graph *gen_grid(int32_t rows, int32_t cols, uint64_t seed, int wmode, uint32_t wparam) {
    int64_t n64 = (int64_t)rows * cols;
    if (rows < 1 || cols < 1 || n64 > 2147483646LL) return NULL;
    int32_t n = (int32_t)n64;
    gen_graph *g = (gen_graph *)calloc(1, sizeof(gen_graph));
    g->n = n;
    g->offsets = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int64_t m = 2LL * ((int64_t)rows * (cols - 1) + (int64_t)(rows - 1) * cols);
    g->m = m;
    g->indices = (int32_t *)malloc((size_t)(m ? m : 1) * sizeof(int32_t));
    g->weights = (uint32_t *)malloc((size_t)(m ? m : 1) * sizeof(uint32_t));
    /* offsets: degree depends on border position */
    int64_t acc = 0;
    for (int32_t r = 0; r < rows; r++)
        for (int32_t c = 0; c < cols; c++) {
            g->offsets[(int64_t)r * cols + c] = (int32_t)acc;
            acc += (r > 0) + (c > 0) + (c < cols - 1) + (r < rows - 1);
        }
    g->offsets[n] = (int32_t)acc;
    uint64_t wseed = seed * 0x100000001B3ULL + 17;
#pragma omp parallel for schedule(static)
    for (int32_t r = 0; r < rows; r++)
        for (int32_t c = 0; c < cols; c++) {
            int32_t v = r * cols + c;
            int64_t o = g->offsets[v];
            int32_t nb[4];
            int k = 0;
            if (r > 0) nb[k++] = v - cols;
            if (c > 0) nb[k++] = v - 1;
            if (c < cols - 1) nb[k++] = v + 1;
            if (r < rows - 1) nb[k++] = v + cols;
            for (int i = 0; i < k; i++) {
                g->indices[o + i] = nb[i];
                g->weights[o + i] = pair_weight(wseed, wmode, wparam, (uint32_t)v, (uint32_t)nb[i]);
            }
        }
    return g;
}

/* R-MAT with probabilities (a,b,c,1-a-b-c) quantised to 16 bits per level. */
gen_graph *gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed, int wmode,
                    uint32_t wparam) {
    if (scale < 1 || scale > 30) return NULL;
    int32_t n = (int32_t)(1u << scale);
    int64_t draws = (int64_t)edge_factor << scale;
    uint32_t *src = (uint32_t *)malloc((size_t)draws * sizeof(uint32_t));
    uint32_t *dst = (uint32_t *)malloc((size_t)draws * sizeof(uint32_t));
    if (!src || !dst) { free(src); free(dst); return NULL; }
    uint32_t tA = (uint32_t)llround(a * 65536.0), tAB = (uint32_t)llround((a + b) * 65536.0),
             tABC = (uint32_t)llround((a + b + c) * 65536.0);
    int words = (scale + 3) / 4;
    uint64_t eseed = seed * 0x9E3779B97F4A7C15ULL + 0x1234567ULL;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < draws; i++) {
        uint32_t u = 0, v = 0;
        int lvl = 0;
        for (int wd = 0; wd < words; wd++) {
            uint64_t h = hkey(eseed, ((uint64_t)i << 4) | (uint64_t)wd);
            for (int k = 0; k < 4 && lvl < scale; k++, lvl++) {
                uint32_t r = (uint32_t)((h >> (16 * k)) & 0xFFFFu);
                uint32_t bit = 1u << (scale - 1 - lvl);
                if (r < tA) {
                } else if (r < tAB) {
                    v |= bit;
                } else if (r < tABC) {
                    u |= bit;
                } else {
                    u |= bit;
                    v |= bit;
                }
            }
        }
        src[i] = u;
        dst[i] = v;
    }
    gen_graph *g = csr_from_pairs(n, draws, src, dst, 1, 1, seed * 0x100000001B3ULL + 29, wmode, wparam);
    free(src);
    free(dst);
    return g;
}

/* G(n, draws): `draws` hashed (u,v) pairs, self-loops dropped, dedup; symmetrised unless directed. */
gen_graph *gen_random(int32_t n, int64_t draws, int directed, uint64_t seed, int wmode, uint32_t wparam) {
    if (n < 1) return NULL;
    uint32_t *src = (uint32_t *)malloc((size_t)(draws ? draws : 1) * sizeof(uint32_t));
    uint32_t *dst = (uint32_t *)malloc((size_t)(draws ? draws : 1) * sizeof(uint32_t));
    uint64_t eseed = seed * 0xD1B54A32D192ED03ULL + 7;
    for (int64_t i = 0; i < draws; i++) {
        uint64_t h = hkey(eseed, (uint64_t)i);
        src[i] = (uint32_t)((h & 0xFFFFFFFFu) % (uint32_t)n);
        dst[i] = (uint32_t)((h >> 32) % (uint32_t)n);
    }
    gen_graph *g = csr_from_pairs(n, draws, src, dst, !directed, 1, seed * 0x100000001B3ULL + 31, wmode, wparam);
    if (g && directed) {
        /* directed graphs: weight per ordered arc, not per pair */
        uint64_t ws = seed * 0x100000001B3ULL + 37;
        for (int32_t v = 0; v < n; v++)
            for (int64_t e = g->offsets[v]; e < g->offsets[v + 1]; e++) {
                uint64_t h = hkey(ws, ((uint64_t)(uint32_t)v << 32) | (uint32_t)g->indices[e]);
                if (wmode == W_UNIFORM) g->weights[e] = 1u + (uint32_t)(h % (uint64_t)wparam);
            }
    }
    free(src);
    free(dst);
    return g;
}

/* ---- random geometric k-nearest-neighbour graph ---- */
typedef struct { double d2; int32_t id; } cand;
static inline int cand_less(cand a, cand b) { return a.d2 < b.d2 || (a.d2 == b.d2 && a.id < b.id); }

gen_graph *gen_rgg_knn(int32_t n, int k, uint64_t seed) {
    if (n < 2 || k < 1 || k > 16) return NULL;
    double *xy = (double *)malloc((size_t)n * 2 * sizeof(double));
    uint64_t ps = seed * 0xA24BAED4963EE407ULL + 3;
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; i++) {
        xy[2 * (int64_t)i] = unit53(hkey(ps, 2ULL * (uint64_t)i));
        xy[2 * (int64_t)i + 1] = unit53(hkey(ps, 2ULL * (uint64_t)i + 1));
    }
    int32_t G = (int32_t)floor(sqrt((double)n / 2.0));
    if (G < 1) G = 1;
    int64_t ncell = (int64_t)G * G;
    int32_t *cell_of = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *cstart = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < n; i++) {
        int32_t cx = (int32_t)(xy[2 * (int64_t)i] * G), cy = (int32_t)(xy[2 * (int64_t)i + 1] * G);
        if (cx >= G) cx = G - 1;
        if (cy >= G) cy = G - 1;
        cell_of[i] = cy * G + cx;
        __atomic_fetch_add(&cstart[cell_of[i] + 1], 1, __ATOMIC_RELAXED);
    }
    for (int64_t cidx = 0; cidx < ncell; cidx++) cstart[cidx + 1] += cstart[cidx];
    int32_t *cpts = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *ccur = (int64_t *)malloc((size_t)ncell * sizeof(int64_t));
    memcpy(ccur, cstart, (size_t)ncell * sizeof(int64_t));
    for (int32_t i = 0; i < n; i++) cpts[ccur[cell_of[i]]++] = i; /* sequential: id order inside a cell */
    free(ccur);
    uint32_t *src = (uint32_t *)malloc((size_t)n * k * sizeof(uint32_t));
    uint32_t *dst = (uint32_t *)malloc((size_t)n * k * sizeof(uint32_t));
    double cs = 1.0 / G;
#pragma omp parallel for schedule(dynamic, 4096)
    for (int32_t p = 0; p < n; p++) {
        cand best[16];
        int nb = 0;
        double px = xy[2 * (int64_t)p], py = xy[2 * (int64_t)p + 1];
        int32_t pcx = cell_of[p] % G, pcy = cell_of[p] / G;
        for (int32_t r = 0; r <= G; r++) {
            for (int32_t dy = -r; dy <= r; dy++) {
                int32_t cy = pcy + dy;
                if (cy < 0 || cy >= G) continue;
                int32_t step = (dy == -r || dy == r) ? 1 : 2 * r;
                for (int32_t dx = -r; dx <= r; dx += (step ? step : 1)) {
                    int32_t cx = pcx + dx;
                    if (cx >= 0 && cx < G) {
                        int64_t cidx = (int64_t)cy * G + cx;
                        for (int64_t t = cstart[cidx]; t < cstart[cidx + 1]; t++) {
                            int32_t q = cpts[t];
                            if (q == p) continue;
                            double ex = px - xy[2 * (int64_t)q], ey = py - xy[2 * (int64_t)q + 1];
                            cand cd = {ex * ex + ey * ey, q};
                            if (nb < k) {
                                int j = nb++;
                                while (j > 0 && cand_less(cd, best[j - 1])) { best[j] = best[j - 1]; j--; }
                                best[j] = cd;
                            } else if (cand_less(cd, best[k - 1])) {
                                int j = k - 1;
                                while (j > 0 && cand_less(cd, best[j - 1])) { best[j] = best[j - 1]; j--; }
                                best[j] = cd;
                            }
                        }
                    }
                    if (r == 0) break;
                }
            }
            double bound = r * cs;
            if (nb == k && best[k - 1].d2 < bound * bound * (1.0 - 1e-12)) break;
            if (nb == n - 1 && nb < k) break;
        }
        for (int j = 0; j < k; j++) {
            src[(int64_t)p * k + j] = (uint32_t)p;
            dst[(int64_t)p * k + j] = (uint32_t)(j < nb ? best[j].id : p); /* p->p dropped as self-loop */
        }
    }
    free(cell_of);
    free(cstart);
    free(cpts);
    gen_graph *g = csr_from_pairs(n, (int64_t)n * k, src, dst, 1, 1, 0, W_CONST, 1);
    free(src);
    free(dst);
    if (!g) { free(xy); return NULL; }
    /* weight = llround(euclidean length * 1e6) + 1, symmetric by (lo,hi) ordering */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int32_t v = 0; v < n; v++)
        for (int64_t e = g->offsets[v]; e < g->offsets[v + 1]; e++) {
            int32_t u = g->indices[e];
            int32_t lo = u < v ? u : v, hi = u < v ? v : u;
            double ex = xy[2 * (int64_t)lo] - xy[2 * (int64_t)hi], ey = xy[2 * (int64_t)lo + 1] - xy[2 * (int64_t)hi + 1];
            g->weights[e] = (uint32_t)(llround(sqrt(ex * ex + ey * ey) * 1e6) + 1);
        }
    g->xy = xy;
    return g;
}

/* CSR from explicit arcs (tests): duplicates keep the MINIMUM weight. */
gen_graph *gen_from_arcs(int32_t n, int64_t cnt, const int32_t *src, const int32_t *dst, const uint32_t *w,
                         int symmetrise) {
    if (n < 1) return NULL;
    int64_t tot = symmetrise ? 2 * cnt : cnt;
    typedef struct { int32_t u, v; uint32_t w; } arc;
    arc *a = (arc *)malloc((size_t)(tot ? tot : 1) * sizeof(arc));
    for (int64_t i = 0; i < cnt; i++) {
        a[i].u = src[i]; a[i].v = dst[i]; a[i].w = w[i];
        if (symmetrise) { a[cnt + i].u = dst[i]; a[cnt + i].v = src[i]; a[cnt + i].w = w[i]; }
    }
    /* counting sort by u then insertion by (v, w) within rows */
    gen_graph *g = (gen_graph *)calloc(1, sizeof(gen_graph));
    g->n = n;
    g->offsets = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    int64_t *st = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < tot; i++) st[a[i].u + 1]++;
    for (int32_t v = 0; v < n; v++) st[v + 1] += st[v];
    arc *s = (arc *)malloc((size_t)(tot ? tot : 1) * sizeof(arc));
    int64_t *cur = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    memcpy(cur, st, ((size_t)n + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < tot; i++) s[cur[a[i].u]++] = a[i];
    free(a);
    g->indices = (int32_t *)malloc((size_t)(tot ? tot : 1) * sizeof(int32_t));
    g->weights = (uint32_t *)malloc((size_t)(tot ? tot : 1) * sizeof(uint32_t));
    int64_t o = 0;
    for (int32_t v = 0; v < n; v++) {
        int64_t b = st[v], e = st[v + 1];
        for (int64_t i = b + 1; i < e; i++) {
            arc x = s[i];
            int64_t j = i - 1;
            while (j >= b && (s[j].v > x.v || (s[j].v == x.v && s[j].w > x.w))) { s[j + 1] = s[j]; j--; }
            s[j + 1] = x;
        }
        g->offsets[v] = (int32_t)o;
        for (int64_t i = b; i < e; i++) {
            if (i > b && s[i].v == s[i - 1].v) continue; /* keep min weight (sorted first) */
            g->indices[o] = s[i].v;
            g->weights[o] = s[i].w;
            o++;
        }
    }
    g->offsets[n] = (int32_t)o;
    g->m = o;
    free(s);
    free(st);
    free(cur);
    return g;
}

int gen_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
