"""Pins for the CPU oracle (-m "not gpu").

The oracle is pinned to things other than itself: hand examples (tests/golden),
an independent brute-force Bellman-Ford, scipy's Dijkstra, closed forms computed
here in plain Python, and theorems of PAPER.md that bound its stepping simulation.
"""
import collections

import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.csgraph

import gen
import oracle
from conftest import golden_value, load_golden, rng_graphs

INF = oracle.INF_INT
SPEC = load_golden("spec_examples.json")


def _graph_from_case(c):
    arcs = np.array(c["arcs"], dtype=np.int64).reshape(-1, 3)
    return gen.from_arcs(c["n"], arcs[:, 0], arcs[:, 1], arcs[:, 2], symmetrise=c.get("symmetrise", False),
                         source=c.get("source", 0), name=c["name"])


# ----------------------------------------------------------------------------- golden
@pytest.mark.parametrize("case", SPEC["sssp"], ids=lambda c: c["name"])
def test_golden_sssp(case):
    g = _graph_from_case(case)
    want = np.array(golden_value(case["dist"]), dtype=np.uint64)
    d, hops = oracle.dijkstra(g, with_hops=True)
    assert (d == want).all()
    if "hops" in case:
        assert hops.tolist() == case["hops"]
        assert oracle.k_n(g) == case["k_n"]
    bf, _ = oracle.bellman_ford(g)
    assert (bf == want).all()
    for pol, par in (("bellman_ford", 0), ("delta", 1), ("delta", 1000), ("rho", 1), ("rho", 2), ("dijkstra", 0)):
        ds, tr, _ = oracle.stepping_sim(g, pol, par)
        assert (ds == want).all(), pol
    if "bf_rounds" in case:
        _, tr, _ = oracle.stepping_sim(g, "bellman_ford")
        assert len(tr) == case["bf_rounds"]
        assert tr["fsize"].tolist() == case["bf_visited_per_round"]
    assert oracle.certify(g, want) == 0


@pytest.mark.parametrize("case", SPEC["csr"], ids=lambda c: c["name"])
def test_golden_csr(case):
    g = _graph_from_case(case)
    assert g.offsets.tolist() == case["offsets"]
    assert g.indices.tolist() == case["targets"]


@pytest.mark.parametrize("case", SPEC["pq"], ids=lambda c: c["name"])
def test_golden_naive_pq(case):
    keys = np.array(case["keys"], dtype=np.uint64)
    q = oracle.NaivePQ(keys)
    q.update(case["updates"])
    out = q.extract(golden_value(case["theta"]))
    assert sorted(out) == case["extracted"]
    assert sorted(q.ids) == case["remaining"]


def test_naive_pq_lazy_update():
    """update, then lower delta, then extract with theta between old and new -> extracted."""
    keys = np.array([10, 10], dtype=np.uint64)
    q = oracle.NaivePQ(keys)
    q.update([0])
    keys[0] = 3
    assert q.extract(5) == {0}


@pytest.mark.parametrize("case", SPEC["select"], ids=lambda c: c["name"])
def test_golden_select(case):
    if "keys" in case:
        keys = np.array(case["keys"], dtype=np.uint64)
    else:
        keys = np.full(case["count"], case["keys_const"], dtype=np.uint64)
    want = golden_value(case["theta"])
    assert oracle.select_exact(keys, case["rho"]) == want
    if case.get("sampled", True):  # the sampled selector only estimates the rho-th key
        for seed in range(5):
            assert oracle.select_sampled(keys, case["rho"], seed=seed) == want


# ----------------------------------------------------------------------------- Dijkstra pins
def test_dijkstra_vs_bruteforce_bellman_ford():
    """>= 200 seeded random graphs (directed and undirected), n <= 2000."""
    graphs = rng_graphs(190, seed0=11, nmax=300) + rng_graphs(12, seed0=12, nmax=2000)
    for g in graphs:
        d = oracle.dijkstra(g)
        bf, passes = oracle.bellman_ford(g)
        assert (d == bf).all(), g.name


def _scipy_dist(g, s):
    a = scipy.sparse.csr_matrix((g.weights.astype(np.float64), g.indices, g.offsets), shape=(g.n, g.n))
    d = scipy.sparse.csgraph.dijkstra(a, directed=True, indices=s)
    out = np.full(g.n, INF, dtype=np.uint64)
    fin = np.isfinite(d)
    out[fin] = d[fin].astype(np.uint64)  # exact: all distances < 2^53
    return out


@pytest.mark.parametrize("name", ["grid64", "rmat12", "rgg64k", "rmat14log"])
def test_dijkstra_vs_scipy_configs(name):
    g = gen.make(name)
    assert (oracle.dijkstra(g) == _scipy_dist(g, g.source)).all()


def test_dijkstra_vs_scipy_random():
    for g in rng_graphs(40, seed0=21, nmax=1500):
        assert (oracle.dijkstra(g) == _scipy_dist(g, g.source)).all()


def test_closed_form_uniform_grid():
    """Uniform weight c on a grid from corner 0: d(r, col) = c * (r + col)."""
    for c in (1, 7, 65535):
        g = gen.grid(23, 31, seed=1, const_weight=c)
        d = oracle.dijkstra(g)
        r, col = np.divmod(np.arange(g.n), 31)
        assert (d == (c * (r + col)).astype(np.uint64)).all()


def _python_bfs(g, s):
    lvl = [-1] * g.n
    lvl[s] = 0
    dq = collections.deque([s])
    while dq:
        u = dq.popleft()
        for e in range(g.offsets[u], g.offsets[u + 1]):
            v = int(g.indices[e])
            if lvl[v] < 0:
                lvl[v] = lvl[u] + 1
                dq.append(v)
    return lvl


def test_closed_form_unit_weights_is_bfs():
    for i, g0 in enumerate(rng_graphs(20, seed0=31, nmax=400)):
        g = gen.random_graph(g0.n, 3 * g0.n, seed=500 + i, directed=bool(i % 2), wmax=1)
        lvl = _python_bfs(g, 0)
        d = oracle.dijkstra(g, 0)
        want = np.array([INF if x < 0 else x for x in lvl], dtype=np.uint64)
        assert (d == want).all()
        assert (oracle.bfs(g, 0) == np.array(lvl)).all()


def test_closed_form_chain_and_star():
    w = np.array([5, 1, 9, 2, 2, 70000], dtype=np.uint32)
    g = gen.chain(7, w, source=0)
    assert oracle.dijkstra(g).tolist() == np.concatenate([[0], np.cumsum(w)]).tolist()
    g = gen.chain(7, w, source=6)
    assert oracle.dijkstra(g).tolist() == np.concatenate([np.cumsum(w[::-1])[::-1], [0]]).tolist()
    lw = np.array([3, 1, 4, 1, 5], dtype=np.uint32)
    g = gen.star(5, lw)
    assert oracle.dijkstra(g, 0).tolist() == [0] + lw.tolist()
    # leaf a to leaf b = w_a + w_b
    d = oracle.dijkstra(g, 3)
    assert d.tolist() == [lw[2]] + [lw[2] + x if i != 2 else 0 for i, x in enumerate(lw)]


def test_closed_form_random_tree_path_sums():
    rs = np.random.default_rng(5)
    for t in range(20):
        n = int(rs.integers(2, 500))
        parent = np.array([0] + [int(rs.integers(0, v)) for v in range(1, n)])
        w = rs.integers(1, 1 << 20, size=n - 1).astype(np.uint32)
        g = gen.from_arcs(n, parent[1:], np.arange(1, n), w, symmetrise=True)
        s = int(rs.integers(0, n))
        # DFS path sums from s over the undirected tree
        want = [None] * n
        want[s] = 0
        stack = [s]
        while stack:
            u = stack.pop()
            for e in range(g.offsets[u], g.offsets[u + 1]):
                v = int(g.indices[e])
                if want[v] is None:
                    want[v] = want[u] + int(g.weights[e])
                    stack.append(v)
        assert oracle.dijkstra(g, s).tolist() == want


def test_large_weights_no_overflow():
    """uint64 arithmetic: a chain of 2^32-1 weights exceeds 2^32 quickly."""
    w = np.full(50, 0xFFFFFFFF, dtype=np.uint32)
    g = gen.chain(51, w)
    d = oracle.dijkstra(g)
    assert int(d[-1]) == 50 * 0xFFFFFFFF
    assert oracle.bellman_ford(g)[0][-1] == d[-1]


def test_hops_tie_break():
    """Hop distance = fewest edges among shortest paths."""
    # 0->1->2->3 (1+1+1) and 0->3 (3): d[3] = 3 with 1 hop
    g = gen.from_arcs(4, [0, 1, 2, 0], [1, 2, 3, 3], [1, 1, 1, 3])
    d, h = oracle.dijkstra(g, 0, with_hops=True)
    assert d.tolist() == [0, 1, 2, 3] and h.tolist() == [0, 1, 2, 1]


# ----------------------------------------------------------------------------- certificate
def test_certificate_accepts_and_rejects():
    g = gen.make("rgg64k")
    d = oracle.dijkstra(g)
    assert oracle.certify(g, d) == 0
    bad = d.copy()
    bad[g.source] = 1
    assert oracle.certify(g, bad)[0] == 1
    v = int(g.indices[g.offsets[g.source]])
    bad = d.copy()
    bad[v] += 1  # too large: the tight in-arc now violates (ii)
    assert oracle.certify(g, bad)[0] == 2
    far = int(np.argmax(np.where(d == oracle.INF, 0, d)))
    bad = d.copy()
    bad[far] -= 1  # too small: no tight in-arc (iii) (far has max distance, so no out-arc breaks (ii))
    assert oracle.certify(g, bad) == (3, far)
    # (iv): an unreachable zero-weight 2-cycle with self-consistent finite labels
    h = gen.from_arcs(4, [0, 2, 3], [1, 3, 2], [1, 0, 0])
    dd = np.array([0, 1, 5, 5], dtype=np.uint64)
    assert oracle.certify(h, dd, source=0) == (4, 2)
    dd[2] = dd[3] = oracle.INF
    assert oracle.certify(h, dd, source=0) == 0


# ----------------------------------------------------------------------------- stepping simulation pins
POLS = [("bellman_ford", 0), ("delta", 1), ("delta", 64), ("delta", 1 << 16), ("rho", 1), ("rho", 4), ("rho", 64),
        ("dijkstra", 0)]


def test_sim_distances_and_theorems_random():
    graphs = rng_graphs(60, seed0=41, nmax=250)
    for g in graphs:
        d, hops = oracle.dijkstra(g, with_hops=True)
        kn = int(hops.max())
        L = g.max_weight
        for pol, par in POLS:
            for warm in (False, True):
                if warm and pol != "rho":
                    continue
                ds, tr, ext = oracle.stepping_sim(g, pol, par, warmup=warm, ext_counts=True)
                assert (ds == d).all(), (g.name, pol, par)
                rounds = len(tr)
                # snapshot semantics: every policy needs >= k_n + 1 rounds
                assert rounds >= kn + 1
                # Lemma num-ext: v extracted at most hops(v) times (source once)
                reach = hops >= 0
                assert (ext[reach] <= np.maximum(hops[reach], 1)).all()
                assert (ext[~reach] == 0).all()
                assert tr["fsize"].sum() == ext.sum()
                if pol == "bellman_ford":
                    assert rounds == kn + 1  # synchronous BF: exactly k_n + 1 rounds
                if pol == "delta":
                    # Thm deltass: steps <= ceil(k_n L / D) + k_n  (+1 final drain round)
                    assert rounds <= -(-kn * L // par) + kn + 1
                if pol == "dijkstra":
                    # one distinct distance value per round
                    assert rounds == len(np.unique(d[reach]))
                # trace consistency: Q_{r+1} = Q_r - F_r + inserts
                q = tr["qsize"]
                assert (q[1:] == q[:-1] - tr["fsize"][:-1] + tr["inserts"][:-1]).all()
                assert q[-1] - tr["fsize"][-1] + tr["inserts"][-1] == 0


def _k_rho(g, rho):
    """Brute force k_rho: min k s.t. for all v, r_rho(v) <= rbar_k(v)."""
    n = g.n
    allpairs = [oracle.dijkstra(g, v, with_hops=True) for v in range(n)]
    for k in range(0, n + 1):
        ok = True
        for v in range(n):
            d, h = allpairs[v]
            fin = d != oracle.INF
            ds = np.sort(d[fin])
            r_rho = int(ds[min(rho, len(ds)) - 1])
            far = fin & (h > k)
            rbar = int(d[far].min()) if far.any() else INF
            if r_rho > rbar:
                ok = False
                break
        if ok:
            return k
    return n


def test_sim_rho_undirected_step_bound():
    """Thm rho-steps-un: exact rho-stepping on an undirected connected graph
    finishes within (2 k_rho + 3) * ceil(n / rho) steps."""
    rs = np.random.default_rng(77)
    checked = 0
    for t in range(40):
        n = int(rs.integers(4, 40))
        g = gen.random_graph(n, 3 * n, seed=900 + t, directed=False, wmax=int(rs.choice([3, 50, 1000])))
        if (oracle.bfs(g, 0) < 0).any():
            continue
        g.source = 0
        for rho in (1, 2, 3, 5, 8):
            if rho > n:
                continue
            kr = _k_rho(g, rho)
            _, tr, _ = oracle.stepping_sim(g, "rho", rho, exact=True)
            assert len(tr) <= (2 * kr + 3) * (-(-n // rho)), (n, rho, kr, len(tr))
            checked += 1
    assert checked > 50


def test_sim_rho_large_equals_bf():
    """|Q| <= rho -> theta = +inf: rho >= n behaves exactly like Bellman-Ford."""
    g = gen.make("grid64")
    _, a, _ = oracle.stepping_sim(g, "rho", g.n)
    _, b, _ = oracle.stepping_sim(g, "bellman_ford")
    assert len(a) == len(b) and (a["fsize"] == b["fsize"]).all() and (a["edges"] == b["edges"]).all()


def test_sim_delta_huge_is_bf():
    """Delta >= n*L: every theta covers all keys, so Delta* = BF."""
    g = gen.make("grid64")
    _, a, _ = oracle.stepping_sim(g, "delta", g.n * 65535)
    _, b, _ = oracle.stepping_sim(g, "bellman_ford")
    assert len(a) == len(b) and (a["fsize"] == b["fsize"]).all()


def test_sim_delta_stepping_pins():
    """Delta-stepping with FinishCheck (Table; reading R19).

    - Distances equal Dijkstra's on random directed and undirected graphs.
    - Delta <= min weight: bucket i holds exactly the vertices at distance i*Delta-ish, so
      every reached vertex is extracted exactly once and the rounds are the distinct
      finite distances (Dijkstra by distance classes).
    - Delta >= n*L: one bucket, refilled by Bellman-Ford substeps, so the trace equals BF.
    """
    for g in rng_graphs(40, seed0=77, nmax=400):
        want = oracle.dijkstra(g)
        for D in (1, 7, 1000, 1 << 40):
            d, tr, ext = oracle.stepping_sim(g, "delta_stepping", D, ext_counts=True)
            assert np.array_equal(d, want), (g.name, D)
    for name in ("grid64", "rmat12"):
        g = gen.make(name)
        want, hops = oracle.dijkstra(g, with_hops=True)
        d, tr, ext = oracle.stepping_sim(g, "delta_stepping", 1, ext_counts=True)
        fin = want != oracle.INF
        assert np.array_equal(d, want)
        assert (ext[fin] == 1).all()
        assert len(tr) == len(np.unique(want[fin]))
        _, a, _ = oracle.stepping_sim(g, "delta_stepping", g.n * (1 << 18))
        _, b, _ = oracle.stepping_sim(g, "bellman_ford")
        assert len(a) == len(b) and (a["fsize"] == b["fsize"]).all()
        assert len(b) == int(hops.max()) + 1


# ----------------------------------------------------------------------------- selection pins
def test_select_sampled_rank_bound():
    """App. cpam: with c = 10 the sampled theta's rank lies within a constant
    factor of rho w.h.p.; SPEC S:351 makes it concrete: rank in [rho/2, 2 rho] in >= 95% of 200 trials."""
    rs = np.random.default_rng(3)
    keys = rs.permutation(np.arange(1, 10001)).astype(np.uint64)
    rho = 1000
    good = 0
    for seed in range(200):
        th = oracle.select_sampled(keys, rho, seed=seed)
        rank = int((keys <= th).sum())
        good += rho // 2 <= rank <= 2 * rho
    assert good >= 190


def test_select_sampled_degenerate():
    keys = np.array([5, 1, 3], dtype=np.uint64)
    assert oracle.select_sampled(keys, 3) == INF  # |Q| <= rho -> drain
    assert oracle.select_sampled(keys, 2) in (1, 3, 5)
    assert oracle.select_sampled(np.full(100, 9, np.uint64), 10, seed=4) == 9


def test_select_exact_is_kth():
    rs = np.random.default_rng(8)
    for t in range(50):
        q = int(rs.integers(2, 3000))
        keys = rs.integers(0, 1 << 40, size=q, dtype=np.uint64)
        rho = int(rs.integers(1, q))
        assert oracle.select_exact(keys, rho) == int(np.sort(keys)[rho - 1])


# ----------------------------------------------------------------------------- bounded Dijkstra (bench sample)
@pytest.mark.parametrize("name", ["rmat12", "grid64", "rgg64k"])
def test_dijkstra_budget(name):
    """The bounded sample bench.py times: with budget >= m it is the full Dijkstra (distances
    equal, every reachable vertex settled once, scanned = the settled vertices' degrees); with a
    smaller budget it stops at the first pop after the budget is reached, every settled vertex
    is exact, and the settled ones are the closest (Dijkstra's pop order)."""
    g = gen.make(name)
    want = oracle.dijkstra(g)
    deg = np.diff(g.offsets.astype(np.int64))
    reach = want != oracle.INF
    scanned, settled, d = oracle.dijkstra_budget(g, g.source, g.m, return_dist=True)
    assert np.array_equal(d, want)
    assert settled == int(reach.sum())
    assert scanned == int(deg[reach].sum())
    order = np.argsort(want[reach], kind="stable")
    dr = deg[reach][order]
    prev = 0
    for b in (1, 7, g.m // 10, g.m // 3, g.m - 1):
        sc, st, d = oracle.dijkstra_budget(g, g.source, b, return_dist=True)
        assert st >= prev
        prev = st
        # stops at the first pop with scanned >= b: the last settled vertex pushed it over
        assert sc >= min(b, scanned) and sc - dr[:st].max(initial=0) < b
        # exactness of what was settled: st vertices of the true distance order carry exact values
        exact = (d == want) & reach
        assert exact.sum() >= st
        # the settled set is the st closest (Dijkstra pops in distance order; ties at the
        # st-th smallest distance kth in any order): it holds every vertex closer than kth and
        # only vertices at most kth away, and scanned is the sum of its degrees
        kth = np.sort(want[reach])[st - 1]
        assert int(deg[reach][want[reach] < kth].sum()) <= sc <= int(deg[reach][want[reach] <= kth].sum())
