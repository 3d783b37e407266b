"""Full-size parity on the five BASELINE.json configurations, in the launch configuration bench.py times.

Every vertex's distance is compared with the oracle's Dijkstra (feasible at these sizes:
~20 s for R-MAT 24 on one host core), and the optimality certificate is checked on the
GPU output as an independent full-size property.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# (policy, param) per config: the bench defaults plus parameters that exercise other paths
CASES = {
    "grid256": [("rho", 1 << 12), ("rho", 1 << 21), ("delta", 1 << 13), ("bellman_ford", 0),
                ("delta_stepping", 1 << 13)],
    "rmat20": [("rho", 1 << 15), ("rho", 1 << 18), ("delta", 1 << 13), ("bellman_ford", 0),
               ("delta_stepping", 1 << 13), ("dijkstra", 0)],
    "rgg4m": [("rho", 1 << 12), ("rho", 1 << 15), ("delta", 1 << 8), ("bellman_ford", 0),
              ("delta_stepping", 1 << 10)],
    "rmat24": [("rho", 360000), ("rho", 1 << 15), ("rho", 1 << 18), ("rho", 1 << 21), ("delta", 1 << 15),
               ("bellman_ford", 0)],
    "grid4096": [("rho", 1 << 12), ("delta", 1 << 13), ("bellman_ford", 0)],
}


@pytest.mark.parametrize("name", list(CASES))
def test_full_config(cuda_device, name):
    import paper_2105_06145_b200 as P

    g = gen.make(name)
    want, hops = oracle.dijkstra(g, with_hops=True)
    kn = int(hops.max())
    h = P.SSSP.from_graph(g, validate=True)
    for pol, par in CASES[name]:
        got = P.dist_to_u64(h.run(g.source, pol, par))
        if not np.array_equal(got, want):
            bad = np.flatnonzero(got != want)
            raise AssertionError(f"{name}/{pol}/{par}: {len(bad)} mismatches, first {bad[0]}: "
                                 f"{got[bad[0]]} vs {want[bad[0]]}")
    assert oracle.certify(g, got) == 0
    # snapshot semantics: BF makes exactly k_n + 1 rounds, every policy at least k_n + 1
    for pol, par in CASES[name][:1] + [("bellman_ford", 0)]:
        got = P.dist_to_u64(h.run(g.source, pol, par, snapshot=True))
        assert np.array_equal(got, want), f"{name}/{pol}/{par}/snapshot"
        assert h.last_stats["rounds"] >= kn + 1
        if pol == "bellman_ford":
            assert h.last_stats["rounds"] == kn + 1


def test_large_id_space(cuda_device):
    """n = 2^27 with the reachable part spread over the whole id range: 64-bit index math
    in the queue, chunk and output paths (ids above 2^26 and near n-1)."""
    import paper_2105_06145_b200 as P

    n = 1 << 27
    rs = np.random.default_rng(27)
    k = 3000
    ids = np.sort(rs.choice(n, size=k, replace=False)).astype(np.int64)
    ids[-1] = n - 1
    src = np.concatenate([ids[:-1], ids[rs.integers(0, k, 4 * k)]])
    dst = np.concatenate([ids[1:], ids[rs.integers(0, k, 4 * k)]])
    w = rs.integers(1, 1 << 20, len(src)).astype(np.uint32)
    keep = src != dst
    g = gen.from_arcs(n, src[keep], dst[keep], w[keep], symmetrise=True, source=int(ids[0]))
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    for pol, par in (("rho", 64), ("delta", 1 << 18), ("bellman_ford", 0), ("delta_stepping", 1 << 18)):
        got = P.dist_to_u64(h.run(g.source, pol, par))
        assert np.array_equal(got, want), pol
    h.close()


TRACE_FIELDS = ["qsize", "fsize", "edges", "inserts", "theta"]
TRACE_CASES = {
    "grid256": [("bellman_ford", 0, {}), ("delta", 1 << 13, {}), ("rho", 1 << 10, dict(exact=True))],
    "rmat20": [("bellman_ford", 0, {}), ("delta", 1 << 15, {}), ("rho", 1 << 15, dict(exact=True)),
               ("rho", 1 << 15, dict(exact=True, warmup=True))],
    "rgg4m": [("delta", 1 << 12, {}), ("rho", 1 << 13, dict(exact=True))],
    "rmat24": [("bellman_ford", 0, {}), ("rho", 1 << 18, dict(exact=True, warmup=True))],
}


@pytest.mark.parametrize("name", list(TRACE_CASES))
def test_full_round_trace_parity(cuda_device, name):
    """At the full BASELINE sizes, per-round |Q_r|, |F_r|, E_r, inserts_r and theta_r of the
    deterministic policies (snapshot rounds, exact rho) equal the oracle's sequential Alg. 1
    simulation, round by round, and the distances equal its Dijkstra."""
    import paper_2105_06145_b200 as P

    g = gen.make(name)
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    for pol, par, kw in TRACE_CASES[name]:
        d, st, tr, _ = h.run(g.source, pol, par, trace_cap=1 << 16, snapshot=True, warmup=kw.get("warmup", False),
                             exact=kw.get("exact", False))
        assert np.array_equal(P.dist_to_u64(d), want), (name, pol, par)
        _, tr_ref, _ = oracle.stepping_sim(g, pol, par, exact=kw.get("exact", True), warmup=kw.get("warmup", False))
        assert st["rounds"] == len(tr_ref), (name, pol, par, st["rounds"], len(tr_ref))
        for f in TRACE_FIELDS:
            if not np.array_equal(tr[f], tr_ref[f]):
                r = int(np.flatnonzero(tr[f] != tr_ref[f])[0])
                raise AssertionError(f"{name}/{pol}/{par} round {r + 1} {f}: gpu {tr[f][r]} oracle {tr_ref[f][r]}")
    h.close()


OPTION_CASES = {
    # run options off the default path, at full size: bidirectional relaxation (all five
    # configs are undirected), other fusion budgets and no fusion, the near/far queue off,
    # snapshot rounds with sampled rho
    "rgg4m": [("delta", 1 << 12, dict(bidir=True)), ("delta", 1 << 13, dict(fuse_budget=256)),
              ("delta", 1 << 12, dict(fuse=False)), ("rho", 1 << 13, dict(nearfar=False))],
    "grid4096": [("delta", 1 << 17, dict(bidir=True)), ("delta", 1 << 18, dict(fuse_budget=256))],
    "rmat24": [("rho", 1 << 18, dict(nearfar=False)), ("rho", 1 << 18, dict(bidir=True)),
               ("rho", 1 << 18, dict(snapshot=True)), ("delta", 1 << 17, dict(bidir=True))],
}


@pytest.mark.parametrize("name", list(OPTION_CASES))
def test_full_options(cuda_device, name):
    import paper_2105_06145_b200 as P

    g = gen.make(name)
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    for pol, par, kw in OPTION_CASES[name]:
        got = P.dist_to_u64(h.run(g.source, pol, par, **kw))
        if not np.array_equal(got, want):
            bad = np.flatnonzero(got != want)
            raise AssertionError(f"{name}/{pol}/{par}/{kw}: {len(bad)} mismatches, first {bad[0]}")
    h.close()
