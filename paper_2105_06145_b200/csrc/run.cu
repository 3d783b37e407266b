// run.cu — the sssp_* handle API: workspace layout, validation kernel, launch of the
// round loop (loop.cuh; kernels instantiated in inst.cu) and result read-back.
#include "loop.cuh"

#include <algorithm>
#include <unordered_map>
#include <vector>

namespace sssp {

// --------------------------------------------------------------------- arc interleave
// arc[e] = {idx[e], w[e]}: the relax reads an arc's head and weight with one 8-byte load,
// so a light vertex's row costs one TLB lookup in one 8m-byte array instead of one in
// each of two 4m-byte arrays (random rows over GBs are TLB-miss bound)
__global__ void interleave_arcs(int64_t m, const int32_t* __restrict__ idx, const uint32_t* __restrict__ w,
                                uint2* __restrict__ arc) {
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gsize)
        arc[e] = make_uint2((uint32_t)idx[e], w[e]);
}

// relabelled arcs: row of new vertex u = old row of old_of_new(u), heads renamed; one warp
// per vertex (create time only)
__global__ void relabel_arcs(int32_t n, const int32_t* __restrict__ off, const int32_t* __restrict__ idx,
                             const uint32_t* __restrict__ w, const int32_t* __restrict__ new_of_old,
                             const int32_t* __restrict__ roff, uint2* __restrict__ arc) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t o = gw; o < n; o += nw) {  // old vertex o -> new row new_of_old[o]
        const int32_t u = new_of_old[o];
        const int32_t b = off[o], deg = off[o + 1] - b, nb = roff[u];
        for (int32_t k = lane; k < deg; k += 32) arc[nb + k] = make_uint2((uint32_t)new_of_old[idx[b + k]], w[b + k]);
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
    uint64_t* ws_dist2;  // second internal distance buffer (batch runs double-buffer)
    Ctrl* ctrl;
    Ctrl* h_ctrl;  // pinned host mirror for result readback
    int device;
    cudaEvent_t ev[2];
    int num_sms;
    int grid[5][2][4];
    int last_block;  // threads per CTA of the last launch (unit-specific)
    // batch runs: a copy stream overlaps the read-back of run i with run i+1
    cudaStream_t copy_stream;
    cudaEvent_t ev_done[2], ev_copied[2];
    struct RunStatus {
        int32_t status;
        int32_t pad;
        int64_t rounds;
    } * h_status;  // pinned, one per run of a batch
    int32_t h_status_cap;
    uint64_t* dint;  // isolated-vertex compaction: the run's internal distance array (new ids)
};

namespace {

struct Layout {
    uint2* arc;  // interleaved {head, weight} copy of the CSR arcs
    // isolated-vertex compaction (may_compact): new offsets, old <-> new ids, distances
    int32_t* roff;
    int32_t* nofo;
    int32_t* ofno;
    uint64_t* dint;
    uint64_t* dist;
    uint64_t* dist2;
    int32_t *q0, *q1;
    int64_t qcap;
    Desc* chunks;
    int64_t ccap;
    int64_t cspill;
    int32_t* counters;
    uint64_t* cta_min;
    int64_t* cta_delta;
    int32_t* cta_ext;
    Desc* light;
    uint64_t* samples;
    Ctrl* ctrl;
    int32_t* err;
    size_t bytes;
};

// Power-law graphs (m >= 20 n, the complement of the fusion rule) often have many
// isolated vertices (47 % of rmat24).  sssp_create then renumbers the others 0..nz-1 in
// their original order and the isolated ones after them, and the run works on the first
// nz ids only: the live part of delta shrinks (134 -> 71 MB on rmat24, below the L2 size).
// The workspace is reserved whenever it may apply; it applies if >= n/16 are isolated.
bool may_compact(int32_t n, int64_t m, uint32_t flags) {
    return !(flags & SSSP_NO_RELABEL) && m >= (int64_t)kSparseDeg * n && n >= 64;
}

Layout carve(void* base, int32_t n, int64_t m, uint32_t flags) {
    Carver c(base);
    Layout L;
    const bool compact = may_compact(n, m, flags);
    // queue: kShards segments of qcap (2x the even share + slack) plus a spill segment of n
    L.qcap = 2 * (((int64_t)n + kShards - 1) / kShards) + 1024;
    const int64_t qlen = kShards * L.qcap + n;
    // chunks per round <= sum over heavy extracted vertices of ceil(deg/kChunk); kernel units
    // built with more arcs per lane (build.py UNIT_DEFINES) cut longer chunks, i.e. fewer
    const int64_t ctot = m / kChunk + std::min<int64_t>(n, m / (kLight + 1)) + 1;
    L.ccap = 2 * ((ctot + kShards - 1) / kShards) + 256;
    L.cspill = ctot;
    const int64_t clen = kShards * L.ccap + ctot;
    L.arc = c.take<uint2>((size_t)m);
    L.ctrl = c.take<Ctrl>(1);
    L.err = c.take<int32_t>(32);
    L.counters = c.take<int32_t>((size_t)3 * 2 * kSeg * kCntStride);
    L.cta_min = c.take<uint64_t>((size_t)3 * kMaxCtas);
    L.cta_delta = c.take<int64_t>((size_t)3 * kMaxCtas);
    L.cta_ext = c.take<int32_t>((size_t)3 * kMaxCtas);
    L.dist = c.take<uint64_t>(n);
    L.dist2 = c.take<uint64_t>(n);
    L.q0 = c.take<int32_t>(qlen);
    L.q1 = c.take<int32_t>(qlen);
    L.chunks = c.take<Desc>(clen);
    L.light = c.take<Desc>(n);
    L.samples = c.take<uint64_t>(kMaxSamples);
    L.roff = compact ? c.take<int32_t>((size_t)n + 1) : nullptr;
    L.nofo = compact ? c.take<int32_t>((size_t)n) : nullptr;
    L.ofno = compact ? c.take<int32_t>((size_t)n) : nullptr;
    L.dint = compact ? c.take<uint64_t>((size_t)n) : nullptr;
    L.bytes = align_up(c.off, 256);
    return L;
}


KernelUnit unit_for(int pol, int mode) {
    const int fuse = mode & 1, bidir = (mode >> 1) & 1;
#define SSSP_UNIT_CASE(P) \
    case P:               \
        return bidir ? (fuse ? kernel_unit_##P##_1_1() : kernel_unit_##P##_1_0()) : (fuse ? kernel_unit_##P##_0_1() : kernel_unit_##P##_0_0());
    switch (pol) {
        SSSP_UNIT_CASE(0)
        SSSP_UNIT_CASE(1)
        SSSP_UNIT_CASE(2)
        SSSP_UNIT_CASE(3)
        SSSP_UNIT_CASE(4)
    }
#undef SSSP_UNIT_CASE
    return KernelUnit{nullptr, nullptr, 0, 0};
}
KernelFn kernel_for(int pol, bool stats, int mode) {
    const KernelUnit u = unit_for(pol, mode);
    return stats ? u.stats : u.plain;
}


// Validate and enqueue one run of the round loop on h->stream (no synchronisation).
sssp_status launch_run(sssp_handle* h, int32_t source, sssp_policy policy, uint64_t param, const sssp_run_opts& o,
                       uint64_t* d_dist_out, int* grid_out, int64_t* max_rounds_out) {
    if (!d_dist_out) return set_error(SSSP_ERR_INVALID, "sssp_run: NULL d_dist_out");
    if (source < 0 || source >= h->n) return set_error(SSSP_ERR_RANGE, "sssp_run: source %d outside [0, %d)", source, h->n);
    if (policy < SSSP_RHO || policy > SSSP_DELTA_STEPPING)
        return set_error(SSSP_ERR_INVALID, "sssp_run: unknown policy %d", (int)policy);
    if ((policy == SSSP_RHO || policy == SSSP_DELTA || policy == SSSP_DELTA_STEPPING) && param == 0)
        return set_error(SSSP_ERR_INVALID, "sssp_run: param (rho / Delta) must be >= 1");
    cudaError_t de = cudaSetDevice(h->device);
    if (de != cudaSuccess) return cuda_error(de, "cudaSetDevice");
    const bool st = (o.flags & SSSP_RUN_STATS) != 0;
    // fusion ("local relaxation within theta"): the paper applies it in its
    // Delta*- and rho-stepping in sparse rounds, average degree below 20
    // (P:1387-1388).  Here the degree rule is per graph (m < 20 n): fusing the low-degree
    // late rounds of R-MAT re-relaxed 17 % more arcs and cost 50 % time (DESIGN.md fusion).
    // Bellman-Ford, Delta-stepping with FinishCheck and Dijkstra never fuse, so their
    // rounds and counters describe those algorithms.
    const bool fu = !(o.flags & (SSSP_RUN_SNAPSHOT | SSSP_RUN_NO_FUSE)) &&
                    (policy == SSSP_RHO || policy == SSSP_DELTA) && h->m < (int64_t)kSparseDeg * h->n;
    RunParams p = h->base;
    if (p.nofo) {  // compacted ids: delta lives in the workspace, the output pass maps it back
        p.dist = h->dint;
        p.out = d_dist_out;
    } else {
        p.dist = d_dist_out;
        p.out = nullptr;
    }
    p.source = source;  // caller's id (the kernel maps it)
    p.param = param;
    p.flags = o.flags;
    p.seed = o.seed;
    p.max_rounds = o.max_rounds > 0 ? o.max_rounds : 4 * (int64_t)h->n + 64;
    p.trace = st ? (sssp_round*)o.d_trace : nullptr;
    p.trace_cap = o.trace_cap;
    p.ext_count = o.d_ext_count;
    // (rho, with its 10-hop depth bound, does best with 96 fused vertices per warp per round:
    // grid4096 -3.8 %, rgg4m -2 %, grid256 -1.5 % against 64; Delta* keeps 64, profiles/r2_depth)
    p.fuse_budget = o.fuse_budget ? (int32_t)o.fuse_budget : (policy == SSSP_RHO ? kFuseBudgetRho : kFuseBudget);
    p.fuse_depth = o.fuse_depth ? (int32_t)std::min<uint32_t>(o.fuse_depth, 1u << 30)
                                : (policy == SSSP_RHO ? kFuseDepthRho : kFuseDepth);
    const int mode = (fu ? 1 : 0) | ((o.flags & SSSP_RUN_BIDIR) ? 2 : 0);
    KernelFn k = kernel_for(policy, st, mode);
    const int grid = h->grid[policy][st][mode];
    void* args[] = {&p};
    cudaError_t e =
        cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(unit_for(policy, mode).block), args, unit_for(policy, mode).smem, h->stream);
    if (e != cudaSuccess) return cuda_error(e, "round-loop launch");
    *grid_out = grid;
    h->last_block = unit_for(policy, mode).block;
    *max_rounds_out = p.max_rounds;
    return SSSP_OK;
}

sssp_status run_status(int32_t status, int64_t max_rounds) {
    if (status == SSSP_ERR_ROUNDS)
        return set_error(SSSP_ERR_ROUNDS, "sssp_run: exceeded max_rounds=%lld", (long long)max_rounds);
    if (status == SSSP_ERR_INTERNAL)
        return set_error(SSSP_ERR_INTERNAL, "sssp_run: an append list overflowed its spill segment (bug)");
    return SSSP_OK;
}

}  // namespace

namespace {

// Isolated-vertex compaction (create time, host + one kernel): non-isolated vertices keep
// their relative order as ids 0..nz-1, isolated ones follow.  The workspace gets the
// renumbered offsets, both id maps and the renumbered arcs; runs map the source in and the
// output pass maps every distance back (launch_run, sssp_round_loop).
cudaError_t build_compaction(sssp_handle* h, const Layout& L, int32_t n, const int32_t* d_offsets,
                             const int32_t* d_indices, const uint32_t* d_weights, int sms, bool* applied) {
    *applied = false;
    std::vector<int32_t> off((size_t)n + 1);
    cudaError_t e = cudaMemcpyAsync(off.data(), d_offsets, off.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                    h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return e;
    int64_t nz = 0;
    for (int32_t v = 0; v < n; v++) nz += off[(size_t)v + 1] > off[v];
    if (n - nz < n / 16) return cudaSuccess;  // too few isolated vertices to pay the output map
    std::vector<int32_t> nofo((size_t)n), ofno((size_t)n), roff((size_t)n + 1);
    int32_t a = 0, b = (int32_t)nz;
    for (int32_t v = 0; v < n; v++) nofo[v] = off[(size_t)v + 1] > off[v] ? a++ : b++;
    for (int32_t v = 0; v < n; v++) ofno[nofo[v]] = v;
    roff[0] = 0;
    for (int32_t u = 0; u < n; u++) roff[(size_t)u + 1] = roff[u] + (off[(size_t)ofno[u] + 1] - off[ofno[u]]);
    e = cudaMemcpyAsync(L.roff, roff.data(), roff.size() * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(L.nofo, nofo.data(), nofo.size() * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(L.ofno, ofno.data(), ofno.size() * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) {
        relabel_arcs<<<sms * 8, 256, 0, h->stream>>>(n, d_offsets, d_indices, d_weights, L.nofo, L.roff, L.arc);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // the host vectors die here
    if (e != cudaSuccess) return e;
    RunParams& p = h->base;
    p.off = L.roff;
    p.n = (int32_t)nz;  // the run's vertices
    p.n_out = n;
    p.nofo = L.nofo;
    p.ofno = L.ofno;
    h->dint = L.dint;
    *applied = true;
    return cudaSuccess;
}

}  // namespace

extern "C" {

size_t sssp_workspace_bytes(int32_t n, int64_t m, uint32_t flags) {
    if (n < 1 || n > 2147483646 || m < 0 || m > 2147483647LL) return 0;
    return carve(nullptr, n, m, flags).bytes;
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

    Layout L = carve(d_workspace, n, m, flags);
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
    h->ws_dist2 = L.dist2;
    h->ctrl = L.ctrl;
    RunParams& b = h->base;
    memset(&b, 0, sizeof(b));
    b.n = n;
    b.m = m;
    b.off = d_offsets;
    b.arc = L.arc;
    b.qbuf[0] = L.q0;
    b.qbuf[1] = L.q1;
    b.qcap = L.qcap;
    b.chunks = L.chunks;
    b.ccap = L.ccap;
    b.cspill = L.cspill;
    b.counters = L.counters;
    b.cta_min = L.cta_min;
    b.cta_delta = L.cta_delta;
    b.cta_ext = L.cta_ext;
    b.light = L.light;
    b.samples = L.samples;
    b.ctrl = L.ctrl;
    for (int pol = 0; pol < kPolicies; pol++)
        for (int st = 0; st < 2; st++)
            for (int sn = 0; sn < 4; sn++) {  // mode: bit 0 fusion, bit 1 bidirectional
                int per_sm = 0;
                const size_t smem = unit_for(pol, sn).smem;
                e = cudaFuncSetAttribute((const void*)kernel_for(pol, st, sn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kernel_for(pol, st, sn),
                                                                      unit_for(pol, sn).block, smem);
                if (e != cudaSuccess || per_sm < 1) {
                    sssp_destroy(h);
                    return e != cudaSuccess ? cuda_error(e, "occupancy query")
                                            : set_error(SSSP_ERR_DEVICE, "round-loop kernel cannot be resident");
                }
                h->grid[pol][st][sn] = std::min(per_sm * sms, kMaxCtas);
            }
    e = cudaMallocHost((void**)&h->h_ctrl, sizeof(Ctrl));
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev[0]);
    if (e == cudaSuccess) e = cudaEventCreate(&h->ev[1]);
    for (int i = 0; i < 2 && e == cudaSuccess; i++) {
        e = cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        sssp_destroy(h);  // every member is value-initialised; destroy null-checks each
        return cuda_error(e, "sssp_create: host resources");
    }
    // control block zeroed once (every run resets what it uses in its prologue)
    e = cudaMemsetAsync(L.ctrl, 0, sizeof(Ctrl), h->stream);
    if (e == cudaSuccess && (flags & SSSP_VALIDATE)) {
        cudaMemsetAsync(L.err, 0, sizeof(int32_t), h->stream);
        validate_csr<<<sms * 4, 256, 0, h->stream>>>(n, m, d_offsets, d_indices, d_weights, L.err);
        e = cudaGetLastError();
        int32_t herr = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, L.err, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess && herr) {
            sssp_destroy(h);
            return set_error(SSSP_ERR_INVALID_GRAPH, "sssp_create: invalid CSR (%s%s%s%s)",
                             (herr & 1) ? "offsets[0]!=0 or offsets[n]!=m " : "", (herr & 2) ? "offsets decrease " : "",
                             (herr & 4) ? "index out of range " : "", (herr & 8) ? "weight < 1" : "");
        }
    }
    bool compacted = false;
    if (e == cudaSuccess && may_compact(n, m, flags))
        e = build_compaction(h, L, n, d_offsets, d_indices, d_weights, sms, &compacted);
    if (e == cudaSuccess && !compacted && m > 0) {
        interleave_arcs<<<sms * 8, 256, 0, h->stream>>>(m, d_indices, d_weights, L.arc);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) {
        sssp_destroy(h);
        return cuda_error(e, "sssp_create");
    }
    *out = h;
    return SSSP_OK;
}

sssp_status sssp_run_ex(sssp_handle* h, int32_t source, sssp_policy policy, uint64_t param,
                        const sssp_run_opts* opts, uint64_t* d_dist_out, sssp_run_stats* stats) {
    if (!h) return set_error(SSSP_ERR_INVALID, "sssp_run: NULL handle");
    sssp_run_opts o;
    memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    int grid = 0;
    int64_t max_rounds = 0;
    cudaEventRecord(h->ev[0], h->stream);
    sssp_status st = launch_run(h, source, policy, param, o, d_dist_out, &grid, &max_rounds);
    if (st != SSSP_OK) return st;
    cudaEventRecord(h->ev[1], h->stream);
    cudaError_t e = cudaMemcpyAsync(&h->h_ctrl->status, &h->ctrl->status, sizeof(Ctrl) - offsetof(Ctrl, status),
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
        stats->dense_scanned = c->tot_dense;
        stats->grid_blocks = grid;
        stats->block_threads = h->last_block;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
        stats->kernel_ms = ms;
    }
    return run_status(c->status, max_rounds);
}

sssp_status sssp_run_batch_host(sssp_handle* h, const int32_t* h_sources, int32_t k, sssp_policy policy,
                                uint64_t param, const sssp_run_opts* opts, uint64_t* h_dist_out,
                                sssp_run_stats* stats) {
    if (!h) return set_error(SSSP_ERR_INVALID, "sssp_run_batch_host: NULL handle");
    if (k < 0 || (k > 0 && (!h_sources || !h_dist_out)))
        return set_error(SSSP_ERR_INVALID, "sssp_run_batch_host: bad batch (k=%d)", k);
    sssp_run_opts o;
    memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    if (o.flags & SSSP_RUN_STATS)
        return set_error(SSSP_ERR_INVALID, "sssp_run_batch_host: SSSP_RUN_STATS is per run (use sssp_run_ex)");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    if (k > h->h_status_cap) {
        if (h->h_status) cudaFreeHost(h->h_status);
        h->h_status = nullptr;
        h->h_status_cap = 0;
        e = cudaMallocHost((void**)&h->h_status, (size_t)k * sizeof(sssp_handle::RunStatus));
        if (e != cudaSuccess) return cuda_error(e, "sssp_run_batch_host: pinned status buffer");
        h->h_status_cap = k;
    }
    uint64_t* buf[2] = {h->ws_dist, h->ws_dist2};
    const size_t bytes = (size_t)h->n * sizeof(uint64_t);
    int grid = 0;
    int64_t max_rounds = 0;
    cudaEventRecord(h->ev[0], h->stream);
    for (int32_t i = 0; i < k; i++) {
        const int b = i & 1;
        if (i >= 2) cudaStreamWaitEvent(h->stream, h->ev_copied[b], 0);  // buffer b read back
        sssp_status st = launch_run(h, h_sources[i], policy, param, o, buf[b], &grid, &max_rounds);
        if (st != SSSP_OK) {
            cudaStreamSynchronize(h->stream);
            cudaStreamSynchronize(h->copy_stream);
            return st;
        }
        cudaMemcpyAsync(&h->h_status[i], &h->ctrl->status, sizeof(sssp_handle::RunStatus), cudaMemcpyDeviceToHost,
                        h->stream);
        cudaEventRecord(h->ev_done[b], h->stream);
        cudaStreamWaitEvent(h->copy_stream, h->ev_done[b], 0);
        cudaMemcpyAsync(h_dist_out + (size_t)i * h->n, buf[b], bytes, cudaMemcpyDeviceToHost, h->copy_stream);
        cudaEventRecord(h->ev_copied[b], h->copy_stream);
    }
    cudaEventRecord(h->ev[1], h->copy_stream);
    e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->copy_stream);
    if (e != cudaSuccess) return cuda_error(e, "sssp_run_batch_host");
    int64_t rounds = 0;
    for (int32_t i = 0; i < k; i++) {
        rounds += h->h_status[i].rounds;
        sssp_status st = run_status(h->h_status[i].status, max_rounds);
        if (st != SSSP_OK) return st;
    }
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->rounds = rounds;
        stats->grid_blocks = grid;
        stats->block_threads = h->last_block;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
        stats->kernel_ms = ms;  // whole batch, read-backs included
    }
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
    for (int i = 0; i < 2; i++) {
        if (h->ev_done[i]) cudaEventDestroy(h->ev_done[i]);
        if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->h_status) cudaFreeHost(h->h_status);
    delete h;
    return SSSP_OK;
}

}  // extern "C"
