// pq.cu — the standalone device LaB-PQ (Table tab:interface P:196-211),
// array-based: a flag bitmap over the id universe plus a compacted
// queue of the flagged ids.  Update sets the flag (test_and_set) and the
// 0->1 winner appends; Extract(theta) reads the keys lazily and packs the
// qualifying ids out, the rest into the other queue buffer.
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "internal.h"

namespace sssp {

struct __align__(128) PQCtrl {
    int32_t size;      // |Q|
    int32_t cnt_out;   // extract: qualifying ids (running)
    int32_t cnt_next;  // extract: remaining ids (running)
    int32_t err;       // latched range error
    unsigned long long minv;   // reduce_min result
    unsigned long long theta;  // select result
    int32_t cnt_q;     // extract with cap < n: qualifying ids counted first
    int32_t res_out;   // extract result: ids written (or, with cap_err, ids that qualify)
    int32_t cap_err;   // extract: more than cap qualified, Q left unchanged
    int32_t done;      // last-CTA ticket of the current grid-wide kernel
};

constexpr int kPQBlock = 256;
constexpr int kSelBlock = 1024;

// The last CTA of a grid to call this returns true (after every CTA's writes before the call
// are visible); it resets the ticket for the next kernel.  Lets one launch finish a reduction
// instead of a follow-up kernel or a host round trip.
__device__ __forceinline__ bool last_cta(int32_t* ticket) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        last = atomicAdd(ticket, 1) == (int32_t)gridDim.x - 1;
        if (last) *ticket = 0;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}

__global__ void pq_update_kernel(const int32_t* __restrict__ ids, int64_t count, int32_t n, uint32_t* bm,
                                 int32_t* queue, PQCtrl* c) {
    const int lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * 32; base < count; base += nwarps * 32) {
        const int64_t i = base + lane;
        bool app = false;
        int32_t id = -1;
        if (i < count) {
            id = ids[i];
            if (id < 0 || id >= n) {
                atomicOr(&c->err, 1);
            } else {
                const uint32_t bit = 1u << (id & 31);
                app = !(atomicOr(bm + (id >> 5), bit) & bit);  // test_and_set
            }
        }
        const int32_t s = warp_append_slot(app, &c->size);
        if (app) queue[s] = id;
    }
}

// CTA-wide sum / min of one value per thread (all threads get the result)
template <typename T, typename Op>
__device__ __forceinline__ T cta_reduce(T x, Op op, T* scratch) {
    for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(kFull, x, o));
    if (lane_id() == 0) scratch[threadIdx.x >> 5] = x;
    __syncthreads();
    x = scratch[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) x = op(x, scratch[w]);
    __syncthreads();
    return x;
}
struct OpAdd {
    __device__ int32_t operator()(int32_t a, int32_t b) const { return a + b; }
};
struct OpMin {
    __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a < b ? a : b; }
};
struct OpMax {
    __device__ uint64_t operator()(uint64_t a, uint64_t b) const { return a > b ? a : b; }
};

// Grid-stride visit of the queued keys with U id loads, then U key gathers, in flight per
// thread (a one-at-a-time loop left one gather in flight per thread: ~85 G keys/s)
template <int U, typename F>
__device__ __forceinline__ void for_keys(const int32_t* __restrict__ queue, const uint64_t* __restrict__ keys, int64_t q,
                                         F f) {
    const int64_t step = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < q; base += step) {
        int32_t id[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            id[u] = i < q ? __ldcs(queue + i) : -1;
        }
        uint64_t k[U];
#pragma unroll
        for (int u = 0; u < U; u++) k[u] = id[u] >= 0 ? ld_cg_u64(keys + id[u]) : 0;
#pragma unroll
        for (int u = 0; u < U; u++)
            if (id[u] >= 0) f(k[u], (int32_t)(base + (int64_t)u * blockDim.x));
    }
}

// extract with cap < n: count the qualifying ids first (one atomic per CTA)
__global__ void __launch_bounds__(kPQBlock) pq_count_kernel(const int32_t* __restrict__ queue,
                                                            const uint64_t* __restrict__ keys, uint64_t theta,
                                                            PQCtrl* c) {
    __shared__ int32_t part[kPQBlock / 32];
    const int32_t q = ld_volatile_i32(&c->size);
    int32_t cnt = 0;
    for_keys<8>(queue, keys, q, [&](uint64_t k, int32_t) { cnt += k <= theta; });
    cnt = cta_reduce(cnt, OpAdd{}, part);
    if (threadIdx.x == 0 && cnt) atomicAdd(&c->cnt_q, cnt);
}

// Extract(theta) in one launch: each CTA owns a contiguous range of the queue, cut into tiles
// of kXBlock * kXItems entries (ids and keys of a tile in registers, kXItems gathers in flight
// per thread); the taken and the kept ids of a tile are counted in shared memory and reserved
// with one atomicAdd each per tile (these same-address atomics bound the call: 1,024-id tiles
// made 14 k of them on a 7 M queue); the last CTA publishes the counts and swaps |Q| (no
// finishing kernel, no host step).  With `check` (cap < n) every CTA first reads the count of
// the counting pass and leaves Q untouched if it exceeds cap (the API's "Q is unchanged" on
// SSSP_ERR_CAPACITY).
constexpr int kXBlock = 512;
constexpr int kXItems = 16;
__global__ void __launch_bounds__(kXBlock) pq_extract_kernel(const int32_t* __restrict__ qcur,
                                                             const uint64_t* __restrict__ keys, uint64_t theta,
                                                             int32_t* out, int32_t* qnext, uint32_t* bm, PQCtrl* c,
                                                             int check, int64_t cap) {
    constexpr int kPQItems = kXItems;
    __shared__ int32_t wt[kXBlock / 32], wk[kXBlock / 32];  // per-warp take / keep counts
    __shared__ int32_t base_t, base_k;
    const int64_t q = ld_volatile_i32(&c->size);
    const bool over = check && (int64_t)ld_volatile_i32(&c->cnt_q) > cap;
    const int lane = lane_id(), wid = threadIdx.x >> 5;
    constexpr int64_t kTile = (int64_t)kXBlock * kXItems;
    const int64_t lo = q * blockIdx.x / gridDim.x, hi = q * (blockIdx.x + 1) / gridDim.x;
    for (int64_t t0 = lo; !over && t0 < hi; t0 += kTile) {
        int32_t id[kPQItems];
        uint32_t take = 0, keep = 0;  // per-item bits
#pragma unroll
        for (int u = 0; u < kPQItems; u++) {  // warp w covers [t0 + w*32*items, ...) in 32-id rows
            const int64_t i = t0 + ((int64_t)wid * kPQItems + u) * 32 + lane;
            id[u] = i < hi ? __ldcs(qcur + i) : -1;
        }
        uint64_t k[kPQItems];
#pragma unroll
        for (int u = 0; u < kPQItems; u++) k[u] = id[u] >= 0 ? ld_cg_u64(keys + id[u]) : 0;
        int32_t nt = 0, nk = 0;
#pragma unroll
        for (int u = 0; u < kPQItems; u++) {
            const bool tk = id[u] >= 0 && k[u] <= theta, kp = id[u] >= 0 && !tk;
            take |= (uint32_t)tk << u;
            keep |= (uint32_t)kp << u;
            nt += __popc(__ballot_sync(kFull, tk));
            nk += __popc(__ballot_sync(kFull, kp));
        }
        if (lane == 0) {
            wt[wid] = nt;
            wk[wid] = nk;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int32_t st = 0, sk = 0;
            for (int w = 0; w < kXBlock / 32; w++) {
                const int32_t a = wt[w], b = wk[w];
                wt[w] = st;
                wk[w] = sk;
                st += a;
                sk += b;
            }
            base_t = st ? atomicAdd(&c->cnt_out, st) : 0;
            base_k = sk ? atomicAdd(&c->cnt_next, sk) : 0;
        }
        __syncthreads();
        int32_t pt = base_t + wt[wid], pk = base_k + wk[wid];
#pragma unroll
        for (int u = 0; u < kPQItems; u++) {
            const bool tk = (take >> u) & 1, kp = (keep >> u) & 1;
            const uint32_t mt = __ballot_sync(kFull, tk), mk = __ballot_sync(kFull, kp);
            if (tk) {
                atomicAnd(bm + (id[u] >> 5), ~(1u << (id[u] & 31)));
                out[pt + __popc(mt & lanemask_lt())] = id[u];
            }
            if (kp) qnext[pk + __popc(mk & lanemask_lt())] = id[u];
            pt += __popc(mt);
            pk += __popc(mk);
        }
        __syncthreads();  // wt / wk / bases are rewritten by the next tile
    }
    if (last_cta(&c->done) && threadIdx.x == 0) {
        if (over) {
            c->res_out = c->cnt_q;
            c->cap_err = 1;
        } else {
            c->res_out = c->cnt_out;
            c->size = c->cnt_next;
        }
        c->cnt_out = 0;
        c->cnt_next = 0;
        c->cnt_q = 0;
    }
}

// min over the queued keys: a partial per CTA, the last CTA reduces them
__global__ void __launch_bounds__(kPQBlock) pq_min_kernel(const int32_t* __restrict__ queue,
                                                          const uint64_t* __restrict__ keys, uint64_t* partial,
                                                          PQCtrl* c) {
    __shared__ uint64_t red[kPQBlock / 32];
    const int32_t q = ld_volatile_i32(&c->size);
    uint64_t mn = kInf;
    for_keys<8>(queue, keys, q, [&](uint64_t k, int32_t) { mn = k < mn ? k : mn; });
    mn = cta_reduce(mn, OpMin{}, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = mn;
    if (last_cta(&c->done)) {
        uint64_t m = kInf;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) m = partial[b] < m ? partial[b] : m;
        m = cta_reduce(m, OpMin{}, red);
        if (threadIdx.x == 0) c->minv = m;
    }
}

// ExtDist of rho-stepping over the queue by sampling, one CTA (reading R5/R6,
// round = 0).
__global__ void __launch_bounds__(kSelBlock) pq_select_kernel(const int32_t* __restrict__ queue,
                                                              const uint64_t* __restrict__ keys, uint64_t rho,
                                                              uint64_t seed, uint32_t mode, uint64_t* samples,
                                                              PQCtrl* c) {
    __shared__ SelectSmem sm;
    const int64_t q = ld_volatile_i32(&c->size);
    uint64_t th;
    if ((uint64_t)q <= rho) {
        th = kInf;
    } else {  // sampled (the exact mode runs on the whole grid: pq_hist_kernel)
        const uint64_t s = sample_count((uint64_t)q, rho);
        for (uint64_t j = threadIdx.x; j < s; j += blockDim.x) {
            const uint64_t r = splitmix64(seed ^ splitmix64(j));  // round 0: (0 << 32) | j
            samples[j] = ld_cg_u64(keys + queue[r % (uint64_t)q]);
        }
        __syncthreads();
        uint64_t k = (rho * s + (uint64_t)q - 1) / (uint64_t)q;
        k = k < 1 ? 1 : (k > s ? s : k);
        th = cta_kth_smallest(ArrayKey{samples}, (int64_t)s, k, sm);
    }
    if (threadIdx.x == 0) c->theta = th;
}

// Exact rho-th smallest over the whole queue with all SMs (SSSP_SELECT_EXACT): MSD radix
// select, 8 bits per pass over the bits where the queue's min and max keys differ.  The first
// kernel gathers the keys once into a contiguous copy (every later pass streams it instead of
// gathering again) and its last CTA sets up the digits; every pass is one grid-wide histogram
// of the keys that match the prefix, whose last CTA picks the bin holding the k-th key.  The
// passes after the answer is known exit at once, so the host enqueues a fixed 8 of them and
// synchronises once.
struct SelState {
    unsigned long long prefix;  // bits above `shift` fixed so far
    unsigned long long k;       // rank (1-based) within the keys matching prefix
    int32_t shift;              // bits still open (0 = done)
    int32_t done;
    uint32_t hist[256];
};

__global__ void __launch_bounds__(kPQBlock) pq_minmax_kernel(const int32_t* __restrict__ queue,
                                                             const uint64_t* __restrict__ keys, uint64_t rho,
                                                             uint64_t* kbuf, uint64_t* partial, PQCtrl* c,
                                                             SelState* st) {
    __shared__ uint64_t red[kPQBlock / 32];
    const int32_t q = ld_volatile_i32(&c->size);
    uint64_t lo = kInf, hi = 0;
    for_keys<8>(queue, keys, q, [&](uint64_t x, int32_t i) {
        __stcs(kbuf + i, x);
        lo = x < lo ? x : lo;
        hi = x > hi ? x : hi;
    });
    lo = cta_reduce(lo, OpMin{}, red);
    hi = cta_reduce(hi, OpMax{}, red);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = lo;
        partial[2 * blockIdx.x + 1] = hi;
    }
    if (!last_cta(&c->done)) return;
    lo = kInf;
    hi = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        lo = partial[2 * b] < lo ? partial[2 * b] : lo;
        hi = partial[2 * b + 1] > hi ? partial[2 * b + 1] : hi;
    }
    lo = cta_reduce(lo, OpMin{}, red);
    hi = cta_reduce(hi, OpMax{}, red);
    for (int b = threadIdx.x; b < 256; b += blockDim.x) st->hist[b] = 0;
    if (threadIdx.x == 0) {
        st->done = 1;
        if ((uint64_t)q <= rho) {
            c->theta = kInf;  // |Q| <= rho: extract everything
        } else if (lo == hi) {
            c->theta = lo;
        } else {
            const int top = 63 - __clzll((long long)(lo ^ hi));  // highest differing bit
            st->prefix = top == 63 ? 0 : (lo >> (top + 1)) << (top + 1);
            st->shift = top + 1;
            st->k = rho;
            st->done = 0;
        }
    }
}

__global__ void __launch_bounds__(kPQBlock) pq_hist_kernel(const uint64_t* __restrict__ kbuf, PQCtrl* c,
                                                           SelState* st) {
    constexpr int kW = kPQBlock / 32;
    __shared__ uint32_t h[kW][256];  // one histogram per warp (fewer same-bin shared atomics)
    if (ld_volatile_i32(&st->done)) return;  // (uniform: written by an earlier kernel)
    const int32_t q = ld_volatile_i32(&c->size);
    const int nb = st->shift >= 8 ? 8 : st->shift, sh = st->shift - nb;
    const uint64_t prefix = st->prefix;
    const uint64_t above = sh + nb >= 64 ? 0 : ~((1ull << (sh + nb)) - 1);
    const int wid = threadIdx.x >> 5;
    for (int b = threadIdx.x; b < kW * 256; b += blockDim.x) (&h[0][0])[b] = 0;
    __syncthreads();
    constexpr int U = 16;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < q; base += step) {
        uint64_t x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t i = base + (int64_t)u * blockDim.x;
            x[u] = i < q ? __ldcs(kbuf + i) : ~prefix;  // (never matches: prefix has zero low bits)
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if ((x[u] & above) == prefix && (base + (int64_t)u * blockDim.x) < q)
                atomicAdd(&h[wid][(x[u] >> sh) & ((1u << nb) - 1)], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kW; w++) t += h[w][b];
        if (t) atomicAdd(&st->hist[b], t);
    }
    if (!last_cta(&c->done)) return;
    // the bin holding the k-th key: the 256 global counts into shared memory in parallel (a
    // serial scan of dependent global loads cost ~30 us), then a short serial scan there
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[0][b] = __ldcg(&st->hist[b]);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t cum = 0;
        int b = 0;
        for (; b < (1 << nb) - 1; b++) {
            const uint32_t hb = h[0][b];
            if (cum + hb >= st->k) break;
            cum += hb;
        }
        st->k -= cum;
        st->prefix |= (uint64_t)b << sh;
        st->shift = sh;
        if (sh == 0) {
            st->done = 1;
            c->theta = st->prefix;
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) st->hist[b] = 0;
}

}  // namespace sssp

using namespace sssp;

struct sssp_pq {
    int32_t n;
    const uint64_t* keys;
    uint32_t* bm;
    int32_t* q[2];
    int cur;
    uint64_t* samples;  // sampled select; also the per-CTA partials of min / minmax
    uint64_t* kbuf;     // exact select: the queued keys, gathered once
    SelState* sel;
    PQCtrl* ctrl;
    PQCtrl* h_ctrl;
    cudaStream_t stream;
    int device;
    int grid;
};

namespace {
struct PQLayout {
    PQCtrl* ctrl;
    uint32_t* bm;
    int32_t *q0, *q1;
    uint64_t* samples;
    uint64_t* kbuf;
    SelState* sel;
    size_t bytes;
};
PQLayout pq_carve(void* base, int32_t n) {
    Carver c(base);
    PQLayout L;
    L.ctrl = c.take<PQCtrl>(1);
    L.bm = c.take<uint32_t>(((size_t)n + 31) / 32);
    L.q0 = c.take<int32_t>(n);
    L.q1 = c.take<int32_t>(n);
    L.samples = c.take<uint64_t>(kMaxSamples);
    L.kbuf = c.take<uint64_t>(n);
    L.sel = c.take<SelState>(1);
    L.bytes = align_up(c.off, 256);
    return L;
}

// read back the control block; report a latched range error
sssp_status pq_sync(sssp_pq* q, const char* what) {
    cudaError_t e = cudaMemcpyAsync(q->h_ctrl, q->ctrl, sizeof(PQCtrl), cudaMemcpyDeviceToHost, q->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(q->stream);
    if (e != cudaSuccess) return cuda_error(e, what);
    if (q->h_ctrl->err) {
        cudaMemsetAsync(&q->ctrl->err, 0, sizeof(int32_t), q->stream);
        return set_error(SSSP_ERR_RANGE, "%s: an earlier sssp_pq_update got an id outside [0, %d)", what, q->n);
    }
    return SSSP_OK;
}
}  // namespace

extern "C" {

size_t sssp_pq_workspace_bytes(int32_t n) {
    if (n < 1 || n > 2147483646) return 0;
    return pq_carve(nullptr, n).bytes;
}

sssp_status sssp_pq_create(int32_t n, const uint64_t* d_keys, void* d_ws, size_t ws_bytes, sssp_stream_t stream,
                           sssp_pq** out) {
    if (!out) return set_error(SSSP_ERR_INVALID, "sssp_pq_create: out is NULL");
    *out = nullptr;
    if (n < 1 || n > 2147483646) return set_error(SSSP_ERR_INVALID, "sssp_pq_create: n=%d outside [1, 2^31-2]", n);
    if (!d_keys || !d_ws) return set_error(SSSP_ERR_INVALID, "sssp_pq_create: NULL pointer");
    if ((uintptr_t)d_ws % 256) return set_error(SSSP_ERR_INVALID, "sssp_pq_create: workspace not 256-byte aligned");
    if (ws_bytes < sssp_pq_workspace_bytes(n))
        return set_error(SSSP_ERR_INVALID, "sssp_pq_create: workspace %zu < required %zu", ws_bytes,
                         sssp_pq_workspace_bytes(n));
    int dev = 0, sms = 0;
    cudaError_t e = bind_device_of(d_ws, &dev);
    if (e != cudaSuccess) return cuda_error(e, "sssp_pq_create: workspace is not device memory");
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    PQLayout L = pq_carve(d_ws, n);
    sssp_pq* q = new sssp_pq();
    q->n = n;
    q->keys = d_keys;
    q->bm = L.bm;
    q->q[0] = L.q0;
    q->q[1] = L.q1;
    q->cur = 0;
    q->samples = L.samples;
    q->kbuf = L.kbuf;
    q->sel = L.sel;
    q->ctrl = L.ctrl;
    q->stream = (cudaStream_t)stream;
    q->grid = sms * 8;  // (<= kMaxSamples / 2: the per-CTA partials live in `samples`)
    q->device = dev;
    e = cudaMallocHost((void**)&q->h_ctrl, sizeof(PQCtrl));
    if (e == cudaSuccess) e = cudaMemsetAsync(L.ctrl, 0, sizeof(PQCtrl), q->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(L.bm, 0, ((size_t)n + 31) / 32 * sizeof(uint32_t), q->stream);
    if (e != cudaSuccess) {
        if (q->h_ctrl) cudaFreeHost(q->h_ctrl);
        delete q;
        return cuda_error(e, "sssp_pq_create");
    }
    *out = q;
    return SSSP_OK;
}

sssp_status sssp_pq_update(sssp_pq* q, const int32_t* d_ids, int64_t count) {
    if (!q) return set_error(SSSP_ERR_INVALID, "sssp_pq_update: NULL queue");
    cudaSetDevice(q->device);
    if (count < 0 || (count > 0 && !d_ids)) return set_error(SSSP_ERR_INVALID, "sssp_pq_update: bad batch");
    if (count == 0) return SSSP_OK;
    int64_t blocks = (count + kPQBlock - 1) / kPQBlock;
    if (blocks > q->grid) blocks = q->grid;
    pq_update_kernel<<<(unsigned)blocks, kPQBlock, 0, q->stream>>>(d_ids, count, q->n, q->bm, q->q[q->cur], q->ctrl);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SSSP_OK : cuda_error(e, "sssp_pq_update");
}

sssp_status sssp_pq_size(sssp_pq* q, int64_t* h_size) {
    if (!q || !h_size) return set_error(SSSP_ERR_INVALID, "sssp_pq_size: NULL argument");
    cudaSetDevice(q->device);
    sssp_status s = pq_sync(q, "sssp_pq_size");
    *h_size = q->h_ctrl->size;
    return s;
}

sssp_status sssp_pq_extract(sssp_pq* q, uint64_t theta, int32_t* d_out, int64_t cap, int64_t* h_count) {
    if (!q || !h_count) return set_error(SSSP_ERR_INVALID, "sssp_pq_extract: NULL argument");
    cudaSetDevice(q->device);
    if (cap < 0 || (cap > 0 && !d_out)) return set_error(SSSP_ERR_INVALID, "sssp_pq_extract: bad output buffer");
    // one launch and one synchronisation: a cap >= n can never overflow (|Q| <= n); a smaller
    // one first counts the qualifying ids and the extract kernel itself refuses to change Q
    // when they exceed cap
    const bool check = cap < (int64_t)q->n;
    if (check) pq_count_kernel<<<q->grid, kPQBlock, 0, q->stream>>>(q->q[q->cur], q->keys, theta, q->ctrl);
    pq_extract_kernel<<<q->grid / 4, kXBlock, 0, q->stream>>>(q->q[q->cur], q->keys, theta, d_out, q->q[q->cur ^ 1],
                                                              q->bm, q->ctrl, check ? 1 : 0, cap);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "sssp_pq_extract");
    // (a range error latched by an earlier update is reported here; this extract still ran)
    sssp_status s = pq_sync(q, "sssp_pq_extract");
    if (s != SSSP_OK && s != SSSP_ERR_RANGE) return s;
    *h_count = q->h_ctrl->res_out;
    if (q->h_ctrl->cap_err) {
        cudaMemsetAsync(&q->ctrl->cap_err, 0, sizeof(int32_t), q->stream);
        return set_error(SSSP_ERR_CAPACITY, "sssp_pq_extract: %d ids qualify, cap %lld", q->h_ctrl->res_out,
                         (long long)cap);
    }
    q->cur ^= 1;
    return s;
}

sssp_status sssp_pq_select(sssp_pq* q, uint64_t rho, uint64_t seed, uint32_t mode, uint64_t* h_theta) {
    if (!q || !h_theta) return set_error(SSSP_ERR_INVALID, "sssp_pq_select: NULL argument");
    cudaSetDevice(q->device);
    if (rho == 0) return set_error(SSSP_ERR_INVALID, "sssp_pq_select: rho must be >= 1");
    if (mode != SSSP_SELECT_SAMPLED && mode != SSSP_SELECT_EXACT)
        return set_error(SSSP_ERR_INVALID, "sssp_pq_select: unknown mode %u", mode);
    cudaError_t e = cudaSuccess;
    if (mode == SSSP_SELECT_EXACT) {
        pq_minmax_kernel<<<q->grid, kPQBlock, 0, q->stream>>>(q->q[q->cur], q->keys, rho, q->kbuf, q->samples, q->ctrl,
                                                              q->sel);
        // (a quarter of the grid: each CTA adds 256 counters and takes the last-CTA ticket with
        // same-address atomics, which dominated a pass at 1,184 CTAs: ~30 us for a 58 MB stream)
        for (int pass = 0; pass < 8; pass++)  // 64-bit keys: at most 8 digits
            pq_hist_kernel<<<q->grid / 4, kPQBlock, 0, q->stream>>>(q->kbuf, q->ctrl, q->sel);
    } else {
        pq_select_kernel<<<1, kSelBlock, 0, q->stream>>>(q->q[q->cur], q->keys, rho, seed, mode, q->samples, q->ctrl);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "sssp_pq_select");
    sssp_status s = pq_sync(q, "sssp_pq_select");
    *h_theta = q->h_ctrl->theta;
    return s;
}

sssp_status sssp_pq_reduce_min(sssp_pq* q, uint64_t* h_min) {
    if (!q || !h_min) return set_error(SSSP_ERR_INVALID, "sssp_pq_reduce_min: NULL argument");
    cudaSetDevice(q->device);
    pq_min_kernel<<<q->grid, kPQBlock, 0, q->stream>>>(q->q[q->cur], q->keys, q->samples, q->ctrl);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "sssp_pq_reduce_min");
    sssp_status s = pq_sync(q, "sssp_pq_reduce_min");
    *h_min = q->h_ctrl->minv;
    return s;
}

sssp_status sssp_pq_queue(sssp_pq* q, int32_t* d_out, int64_t cap, int64_t* h_count) {
    if (!q || !h_count) return set_error(SSSP_ERR_INVALID, "sssp_pq_queue: NULL argument");
    cudaSetDevice(q->device);
    sssp_status s = pq_sync(q, "sssp_pq_queue");
    if (s != SSSP_OK) return s;
    const int64_t sz = q->h_ctrl->size;
    *h_count = sz;
    if (sz > cap) return set_error(SSSP_ERR_CAPACITY, "sssp_pq_queue: |Q| = %lld > cap %lld", (long long)sz, (long long)cap);
    if (sz == 0) return SSSP_OK;
    if (!d_out) return set_error(SSSP_ERR_INVALID, "sssp_pq_queue: NULL d_out");
    cudaError_t e = cudaMemcpyAsync(d_out, q->q[q->cur], (size_t)sz * sizeof(int32_t), cudaMemcpyDeviceToDevice, q->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(q->stream);
    return e == cudaSuccess ? SSSP_OK : cuda_error(e, "sssp_pq_queue");
}

sssp_status sssp_pq_destroy(sssp_pq* q) {
    if (!q) return SSSP_OK;
    if (q->h_ctrl) cudaFreeHost(q->h_ctrl);
    delete q;
    return SSSP_OK;
}

}  // extern "C"
