"""GPU parity: sssp_run (the persistent round loop) vs the CPU oracle, through the C ABI.

Distances must match the oracle's Dijkstra bit-exactly (integer arithmetic).  For the
deterministic policies (Bellman-Ford, Delta*, exact rho, Dijkstra) the per-round trace
(|Q_r|, |F_r|, E_r, inserts_r, theta_r) must equal the oracle's stepping simulation
exactly (snapshot semantics, reading R8).
"""
import numpy as np
import pytest

import gen
import oracle
from conftest import golden_value, load_golden, rng_graphs

pytestmark = pytest.mark.gpu

INF = oracle.INF_INT
SPEC = load_golden("spec_examples.json")


def _P():
    import paper_2105_06145_b200 as P

    return P


def _run(h, g, pol, par, **kw):
    P = _P()
    return P.dist_to_u64(h.run(g.source, pol, par, **kw))


def _assert_same(got, want, label):
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        v = int(bad[0])
        raise AssertionError(f"{label}: {len(bad)} mismatches; vertex {v} got {got[v]} want {want[v]}")


SMALL_POLICIES = [("rho", 1), ("rho", 3), ("rho", 64), ("rho", 1 << 21), ("delta", 1), ("delta", 77),
                  ("delta", 4096), ("delta", 1 << 30), ("bellman_ford", 0), ("dijkstra", 0),
                  ("delta_stepping", 1), ("delta_stepping", 977), ("delta_stepping", 1 << 30)]


def test_golden_examples(cuda_device):
    P = _P()
    for c in SPEC["sssp"]:
        arcs = np.array(c["arcs"]).reshape(-1, 3)
        g = gen.from_arcs(c["n"], arcs[:, 0], arcs[:, 1], arcs[:, 2], symmetrise=True, source=c["source"])
        want = np.array(golden_value(c["dist"]), dtype=np.uint64)
        h = P.SSSP.from_graph(g, validate=True)
        for pol, par in SMALL_POLICIES:
            for snap in (False, True):
                _assert_same(_run(h, g, pol, par, snapshot=snap), want, f"{c['name']}/{pol}/{par}/snap{snap}")
        if "bf_rounds" in c:
            _, st, tr, _ = h.run(g.source, "bellman_ford", 0, trace_cap=64, snapshot=True)
            assert st["rounds"] == c["bf_rounds"]
            assert tr["fsize"].tolist() == c["bf_visited_per_round"]


@pytest.mark.parametrize("name", ["grid64", "rmat12", "rgg64k", "rmat14log", "grid256"])
def test_configs_small_all_policies(cuda_device, name):
    P = _P()
    g = gen.make(name)
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g, validate=True)
    for pol, par in SMALL_POLICIES + [("rho", 1 << 10), ("rho", 1 << 15)]:
        for snap in (False, True):
            got = _run(h, g, pol, par, snapshot=snap)
            _assert_same(got, want, f"{name}/{pol}/{par}/snap{snap}")
    for pol, par in (("rho", 256), ("rho", 4096)):
        _assert_same(_run(h, g, pol, par, exact=True), want, f"{name}/{pol}/{par}/exact")
        _assert_same(_run(h, g, pol, par, warmup=False), want, f"{name}/{pol}/{par}/nowarm")
        _assert_same(_run(h, g, pol, par, exact=True, snapshot=True), want, f"{name}/{pol}/{par}/exact/snap")


def test_random_graphs(cuda_device):
    P = _P()
    for g in rng_graphs(60, seed0=101, nmax=3000):
        want = oracle.dijkstra(g)
        h = P.SSSP.from_graph(g)
        for pol, par in (("rho", 2), ("rho", 100), ("delta", 1000), ("bellman_ford", 0), ("dijkstra", 0)):
            for snap in (False, True):
                _assert_same(_run(h, g, pol, par, snapshot=snap), want, f"{g.name}/src{g.source}/{pol}/{par}/{snap}")


def test_edge_cases(cuda_device):
    P = _P()
    # n = 1, m = 0
    g = gen.from_arcs(1, [], [], [])
    h = P.SSSP.from_graph(g)
    for pol, par in SMALL_POLICIES:
        assert _run(h, g, pol, par).tolist() == [0]
    # isolated source in a larger graph
    g = gen.from_arcs(5, [1, 2], [2, 3], [4, 4], symmetrise=True, source=0)
    h = P.SSSP.from_graph(g)
    assert _run(h, g, "rho", 2).tolist() == [0, INF, INF, INF, INF]
    # self-loops and parallel arcs in a user CSR are accepted (reading R11)
    off = np.array([0, 3, 4, 4], np.int32)
    idx = np.array([0, 1, 1, 2], np.int32)
    w = np.array([5, 9, 2, 1], np.uint32)
    g = gen.Graph(n=3, m=4, offsets=off, indices=idx, weights=w, source=0)
    h = P.SSSP.from_graph(g, validate=True)
    for pol, par in SMALL_POLICIES:
        assert _run(h, g, pol, par).tolist() == [0, 2, 3]
    # maximum weights: distances beyond 2^32
    g = gen.chain(300, np.full(299, 0xFFFFFFFF, np.uint32))
    h = P.SSSP.from_graph(g)
    for pol, par in (("rho", 7), ("delta", 1 << 40), ("bellman_ford", 0)):
        d = _run(h, g, pol, par)
        assert int(d[-1]) == 299 * 0xFFFFFFFF
    # a vertex of degree > 64 * 256 (heavy path, many chunks) plus light vertices
    rs = np.random.default_rng(4)
    n = 30000
    src = np.concatenate([np.zeros(n - 1, np.int64), rs.integers(0, n, 40000)])
    dst = np.concatenate([np.arange(1, n), rs.integers(0, n, 40000)])
    wt = rs.integers(1, 1000, len(src)).astype(np.uint32)
    g = gen.from_arcs(n, src, dst, wt, symmetrise=True, source=int(rs.integers(1, n)))
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    for pol, par in SMALL_POLICIES:
        for snap in (False, True):
            _assert_same(_run(h, g, pol, par, snapshot=snap), want, f"hub/{pol}/{par}/snap{snap}")


def test_errors(cuda_device):
    P = _P()
    g = gen.make("grid64")
    h = P.SSSP.from_graph(g)
    with pytest.raises(P.SSSPError) as e:
        h.run(g.n, "rho", 4)
    assert e.value.status == P.SSSP_ERR_RANGE
    with pytest.raises(P.SSSPError) as e:
        h.run(-1, "bellman_ford", 0)
    assert e.value.status == P.SSSP_ERR_RANGE
    for pol in ("rho", "delta"):
        with pytest.raises(P.SSSPError) as e:
            h.run(0, pol, 0)
        assert e.value.status == P.SSSP_ERR_INVALID
    with pytest.raises(P.SSSPError) as e:
        h.run(0, "bellman_ford", 0, max_rounds=3)
    assert e.value.status == P.SSSP_ERR_ROUNDS
    # SSSP_VALIDATE rejects malformed graphs
    import torch

    for bad in ("weight0", "index", "offsets"):
        off = torch.tensor(g.offsets, device="cuda")
        idx = torch.tensor(g.indices, device="cuda")
        w = torch.tensor(g.weights.view(np.int32), device="cuda")
        if bad == "weight0":
            w[5] = 0
        elif bad == "index":
            idx[7] = g.n
        else:
            off[10] = off[12] + 1
        with pytest.raises(P.SSSPError) as e:
            P.SSSP(off, idx, w, validate=True)
        assert e.value.status == P.SSSP_ERR_INVALID_GRAPH


def test_create_failure_loop_releases(cuda_device):
    """sssp_create's failure paths release the handle's stream and events (sssp_destroy on
    every error return): 200 rejected creates leave device memory where it was and a valid
    handle still works afterwards."""
    import torch

    P = _P()
    g = gen.make("grid64")
    off = torch.tensor(g.offsets, device="cuda")
    idx = torch.tensor(g.indices, device="cuda")
    w = torch.tensor(g.weights.view(np.int32), device="cuda")
    w[5] = 0
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(200):
        with pytest.raises(P.SSSPError) as e:
            P.SSSP(off, idx, w, validate=True)
        assert e.value.status == P.SSSP_ERR_INVALID_GRAPH
    torch.cuda.synchronize()
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (64 << 20), f"device memory dropped by {(free0 - free1) >> 20} MiB over 200 failed creates"
    h = P.SSSP.from_graph(g)
    _assert_same(P.dist_to_u64(h.run(g.source, "delta", 4096)), oracle.dijkstra(g), "after failed creates")
    h.close()


TRACE_FIELDS = ["qsize", "fsize", "edges", "inserts", "theta"]


@pytest.mark.parametrize("name", ["grid64", "rmat12", "rgg64k", "rmat14log"])
def test_round_trace_parity(cuda_device, name):
    """Per-round |Q|, |F|, E, inserts and theta equal the oracle's Alg. 1 simulation."""
    P = _P()
    g = gen.make(name)
    d_ref, hops = oracle.dijkstra(g, with_hops=True)
    kn = int(hops.max())
    h = P.SSSP.from_graph(g)
    cases = [("bellman_ford", 0, {}), ("delta", 1000, {}), ("delta", 20000, {}), ("dijkstra", 0, {}),
             ("delta_stepping", 1, {}), ("delta_stepping", 3000, {}),
             ("rho", 64, dict(exact=True, warmup=False)), ("rho", 2048, dict(exact=True, warmup=False)),
             ("rho", 512, dict(exact=True, warmup=True)), ("rho", 16, dict(exact=True, warmup=False)),
             ("rho", 64, dict(exact=True, warmup=False, nearfar=False))]
    for pol, par, kw in cases:
        d, st, tr, ext = h.run(g.source, pol, par, trace_cap=1 << 16, ext_counts=True, snapshot=True, **kw)
        d = P.dist_to_u64(d)
        _assert_same(d, d_ref, f"{name}/{pol}/{par}")
        _, tr_ref, ext_ref = oracle.stepping_sim(g, pol, par, exact=kw.get("exact", True),
                                                 warmup=kw.get("warmup", False), ext_counts=True)
        assert st["rounds"] == len(tr_ref), (pol, par, st["rounds"], len(tr_ref))
        for f in TRACE_FIELDS:
            if not np.array_equal(tr[f], tr_ref[f]):
                r = int(np.flatnonzero(tr[f] != tr_ref[f])[0])
                raise AssertionError(f"{name}/{pol}/{par} round {r + 1} {f}: gpu {tr[f][r]} oracle {tr_ref[f][r]}")
        _assert_same(ext.cpu().numpy(), ext_ref, f"{name}/{pol}/{par} extraction counts")
        assert st["extracted"] == tr_ref["fsize"].sum() and st["edges"] == tr_ref["edges"].sum()
        if pol == "bellman_ford":
            assert st["rounds"] == kn + 1


def test_sampled_rho_invariants(cuda_device):
    """Sampled theta depends on queue order, so only invariants are compared (snapshot
    semantics for the round bounds; live rounds only keep the queue identities)."""
    P = _P()
    g = gen.make("rmat12")
    d_ref, hops = oracle.dijkstra(g, with_hops=True)
    kn = int(hops.max())
    h = P.SSSP.from_graph(g)
    for rho in (16, 256, 4096):
        for seed in range(3):
            d, st, tr, ext = h.run(g.source, "rho", rho, seed=seed, trace_cap=4096, ext_counts=True)
            _assert_same(P.dist_to_u64(d), d_ref, f"rho{rho}/seed{seed}/live")
            q = tr["qsize"]
            assert (q[1:] == q[:-1] - tr["fsize"][:-1] + tr["inserts"][:-1]).all()
            assert q[-1] - tr["fsize"][-1] + tr["inserts"][-1] == 0
            d, st, tr, ext = h.run(g.source, "rho", rho, seed=seed, trace_cap=4096, ext_counts=True, snapshot=True)
            _assert_same(P.dist_to_u64(d), d_ref, f"rho{rho}/seed{seed}")
            assert st["rounds"] >= kn + 1
            reach = hops >= 0
            e = ext.cpu().numpy()
            assert (e[reach] <= np.maximum(hops[reach], 1)).all()  # Lemma num-ext
            q = tr["qsize"]
            assert (q[1:] == q[:-1] - tr["fsize"][:-1] + tr["inserts"][:-1]).all()
            # |Q| <= rho rounds drain the queue (theta = INF)
            small = q <= rho
            assert (tr["theta"][small] == INF).all() and (tr["fsize"][small] == q[small]).all()


@pytest.mark.parametrize("name,rhos", [("rmat20", (1 << 12, 1 << 15)), ("rgg1m", (1 << 10, 1 << 13))])
def test_in_loop_theta_quality(cuda_device, name, rhos):
    """The in-loop sampled theta_r lands near the rho-th smallest key of Q_r (App. cpam,
    P:1928-1933: rank within [rho/2, 2 rho] w.h.p.).  In snapshot rounds Extract deletes
    exactly the keys <= theta_r before any relax, so |F_r| = #{v in Q_r : delta[v] <= theta_r}
    = rank(theta_r); with near/far on, the near part holds Q's rho smallest keys (R18), so the
    rank is over all of Q either way.  Warm-up off (rho_eff = rho in every round)."""
    P = _P()
    g = gen.make(name)
    d_ref = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    for rho in rhos:
        for nearfar in (True, False):
            for seed in range(2):
                d, st, tr, _ = h.run(g.source, "rho", rho, seed=seed, trace_cap=1 << 16, snapshot=True,
                                     warmup=False, nearfar=nearfar)
                _assert_same(P.dist_to_u64(d), d_ref, f"{name}/rho{rho}/nf{nearfar}/seed{seed}")
                big = tr["qsize"] > rho  # rounds that sample (|Q| <= rho drains)
                f = tr["fsize"][big]
                assert len(f) >= 3, f"{name}/rho{rho}: only {len(f)} sampled rounds"
                ok = (f >= rho // 2) & (f <= 2 * rho)
                assert ok.mean() >= 0.95, (f"{name}/rho{rho}/nf{nearfar}/seed{seed}: rank(theta_r) in [rho/2, 2rho] "
                                           f"in {ok.sum()}/{len(f)} rounds; ranks {f[~ok][:10]}")


def test_determinism_and_run_host(cuda_device):
    import torch

    P = _P()
    g = gen.make("rmat14log")
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    outs = [_run(h, g, "rho", 512, seed=s) for s in range(10)]
    for o in outs:
        _assert_same(o, want, "repeat")
    host = torch.empty(g.n, dtype=torch.int64, pin_memory=True)
    h.run_host(g.source, "rho", 512, host)
    _assert_same(host.numpy().view(np.uint64), want, "run_host")
    # a handle on a non-default stream
    s = torch.cuda.Stream()
    off = torch.from_numpy(g.offsets).cuda()
    idx = torch.from_numpy(g.indices).cuda()
    w = torch.from_numpy(g.weights.view(np.int32)).cuda()
    h2 = P.SSSP(off, idx, w, stream=s)
    d = h2.run(g.source, "delta", 1 << 14)
    s.synchronize()
    _assert_same(P.dist_to_u64(d), want, "side stream")


def test_fusion_variants(cuda_device):
    """Fusion (local relaxation within theta) on sparse graphs: any budget,
    or none, gives the oracle's distances; the per-round |Q| identity still holds."""
    P = _P()
    for name in ("grid64", "rgg64k"):
        g = gen.make(name)
        want = oracle.dijkstra(g)
        h = P.SSSP.from_graph(g)
        for pol, par in (("rho", 64), ("rho", 4096), ("delta", 3000), ("delta_stepping", 3000), ("bellman_ford", 0)):
            for kw in (dict(fuse=False), dict(fuse_budget=1), dict(fuse_budget=32), dict(fuse_budget=100000)):
                d, st, tr, _ = h.run(g.source, pol, par, trace_cap=1 << 16, **kw)
                _assert_same(P.dist_to_u64(d), want, f"{name}/{pol}/{par}/{kw}")
                q = tr["qsize"]
                assert (q[1:] == q[:-1] - tr["fsize"][:-1] + tr["inserts"][:-1]).all()
        # fusion must cut the rounds of a high-diameter graph
        h.run(g.source, "rho", 64, fuse=False)
        r0 = h.last_stats["rounds"]
        h.run(g.source, "rho", 64, fuse_budget=4096)
        assert h.last_stats["rounds"] < r0


def test_bidirectional_undirected(cuda_device):
    """Bidirectional relaxation (SURVEY f-2) on undirected graphs: exact
    distances for every policy and mode, including fusion and snapshot rounds."""
    P = _P()
    graphs = [gen.make(n) for n in ("grid64", "rmat12", "rgg64k", "rmat14log")]
    graphs += [g for g in rng_graphs(30, seed0=505, nmax=2000, directed=False)]
    for g in graphs:
        want = oracle.dijkstra(g)
        h = P.SSSP.from_graph(g)
        for pol, par in (("rho", 2), ("rho", 256), ("delta", 1000), ("delta_stepping", 1000), ("bellman_ford", 0),
                         ("dijkstra", 0)):
            for kw in (dict(), dict(snapshot=True), dict(fuse=False)):
                _assert_same(_run(h, g, pol, par, bidir=True, **kw), want, f"{g.name}/{pol}/{par}/{kw}/bidir")


def test_batch_host(cuda_device):
    """sssp_run_batch_host: k sources, each result read back to host while the next runs."""
    P = _P()
    for name in ("rmat14log", "grid64"):
        g = gen.make(name)
        h = P.SSSP.from_graph(g)
        rs = np.random.default_rng(9)
        sources = [g.source] + [int(x) for x in rs.integers(0, g.n, 6)]
        for pol, par in (("rho", 256), ("delta", 5000), ("bellman_ford", 0)):
            out = h.run_batch_host(sources, pol, par).numpy().view(np.uint64)
            for i, s in enumerate(sources):
                _assert_same(out[i], oracle.dijkstra(g, s), f"{name}/{pol}/batch{i}")
        assert h.run_batch_host([], "rho", 4).shape[0] == 0
        with pytest.raises(P.SSSPError):
            h.run_batch_host([0, g.n], "rho", 4)


def test_unaligned_output_buffer(cuda_device):
    """d_dist_out need only be 8-byte aligned (it is the delta array every kernel phase reads,
    including the near/far dense pass): 16- and 8-byte aligned views give the same result."""
    import torch

    P = _P()
    g = gen.make("rmat14log")
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    base = torch.empty(g.n + 2, dtype=torch.int64, device="cuda")
    for off in (0, 1):  # 16-byte and 8-byte aligned views of the same buffer
        out = base[off:off + g.n]
        assert (out.data_ptr() % 16 == 0) == (off == 0)
        for par in (64, 1024):
            h.run(g.source, "rho", par, out=out)
            _assert_same(P.dist_to_u64(out), want, f"offset {off}/rho {par}")
            _, st, _, _ = h.run(g.source, "rho", par, out=out, stats=True)
            assert st["dense_scanned"] > 0  # the dense pass ran
            _assert_same(P.dist_to_u64(out), want, f"offset {off}/rho {par}/stats")


def test_compacted_output_ragged_tail(cuda_device):
    """The compacted runs' output pass maps 512 caller ids per warp step and finishes the ragged
    tail (n mod 512) one id per thread: a dense graph over the first 2,600 of n = 3,001 ids (the
    rest isolated, so the compaction applies and the tail holds isolated vertices), with a
    16- and an 8-byte aligned output array, against the oracle."""
    import torch

    P = _P()
    rs = np.random.default_rng(77)
    n, k = 3001, 2600
    src = rs.integers(0, k, 80000)
    dst = rs.integers(0, k, 80000)
    w = rs.integers(1, 1 << 12, 80000).astype(np.uint32)
    g = gen.from_arcs(n, src, dst, w, symmetrise=True, source=5)
    deg = np.diff(g.offsets.astype(np.int64))
    assert g.m >= 20 * g.n and int((deg == 0).sum()) >= g.n // 16 and g.n % 512 != 0
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    base = torch.empty(g.n + 2, dtype=torch.int64, device="cuda")
    for off in (0, 1):
        out = base[off:off + g.n]
        for pol, par in (("rho", 64), ("bellman_ford", 0), ("delta", 256)):
            out.fill_(-7)
            h.run(g.source, pol, par, out=out)
            _assert_same(P.dist_to_u64(out), want, f"ragged tail offset {off} {pol}")


def test_isolated_vertex_compaction(cuda_device):
    """Power-law graphs with many isolated vertices are renumbered inside the handle (the
    non-isolated ones become 0..nz-1); sources map in and distances / extraction counts map
    back, so results are identical with the compaction on and off, for isolated and
    non-isolated sources."""
    P = _P()
    g = gen.make("rmat14log")
    deg = np.diff(g.offsets.astype(np.int64))
    iso = np.flatnonzero(deg == 0)
    assert g.m >= 20 * g.n and len(iso) >= g.n // 16  # compaction applies
    nz = np.flatnonzero(deg > 0)
    h_on = P.SSSP.from_graph(g)
    h_off = P.SSSP.from_graph(g, relabel=False)
    assert h_on.workspace.numel() > h_off.workspace.numel()
    for s in [int(g.source), int(nz[len(nz) // 2]), int(nz[-1]), int(iso[0]), int(iso[-1])]:
        want = oracle.dijkstra(g, source=s)
        for pol, par, kw in (("rho", 256, {}), ("delta", 1 << 14, {}), ("bellman_ford", 0, dict(snapshot=True)),
                             ("rho", 64, dict(bidir=True)), ("dijkstra", 0, {}), ("delta_stepping", 1 << 12, {}),
                             ("rho", 32, dict(exact=True, snapshot=True, nearfar=False))):
            d_on, st_on, _, e_on = h_on.run(s, pol, par, ext_counts=True, stats=True, **kw)
            d_off, st_off, _, e_off = h_off.run(s, pol, par, ext_counts=True, stats=True, **kw)
            _assert_same(P.dist_to_u64(d_on), want, f"compaction on s={s} {pol}")
            _assert_same(P.dist_to_u64(d_off), want, f"compaction off s={s} {pol}")
            if kw.get("snapshot"):  # deterministic rounds: identical extraction counts per vertex
                _assert_same(e_on.cpu().numpy(), e_off.cpu().numpy(), f"ext counts s={s}")
                assert st_on["rounds"] == st_off["rounds"]
