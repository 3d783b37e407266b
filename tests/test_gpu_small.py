"""GPU parity of the small-frontier rounds: while |Q| <= 1024 and a round's
frontier has <= 32768 arcs, CTA 0 runs the rounds alone and hands them back to the grid.

Every hand-over direction is exercised: entry at round 1, exit because |Q| outgrew the
shared-memory queue, exit because a frontier was too large (the round is undone and re-run by
the grid), re-entry after a grid round, termination inside the small rounds, and max_rounds
exceeded inside them.  Distances must equal the oracle's Dijkstra with the path on and off,
and in snapshot mode the per-round trace must still equal the oracle's Alg. 1 simulation.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

POLICIES = [("bellman_ford", 0, {}), ("delta", 1000, {}), ("delta", 70000, {}), ("dijkstra", 0, {}),
            ("delta_stepping", 3000, {}), ("rho", 64, dict(exact=True, warmup=False)),
            ("rho", 512, dict(exact=True, warmup=True)), ("rho", 1, {}), ("rho", 4096, {})]
TRACE_FIELDS = ["qsize", "fsize", "edges", "inserts", "theta"]


def hub_chain(n_chain=3000, leaves=40000, seed=7):
    """A weighted chain with a hub of `leaves` pendant vertices half way and a second chain
    hanging off the last leaf: small rounds, a frontier too large for one SM, a queue too
    large for shared memory, then small rounds again."""
    rs = np.random.default_rng(seed)
    n = n_chain + leaves + n_chain
    hub = n_chain // 2
    src = list(range(n_chain - 1)) + [hub] * leaves + [n_chain + leaves - 1] + \
        list(range(n_chain + leaves, n - 1))
    dst = list(range(1, n_chain)) + list(range(n_chain, n_chain + leaves)) + [n_chain + leaves] + \
        list(range(n_chain + leaves + 1, n))
    w = rs.integers(1, 1000, len(src))
    return gen.from_arcs(n, np.array(src), np.array(dst), w, symmetrise=True, source=0)


def _trace_same(g, tr, st, pol, par, kw, label):
    _, tr_ref, _ = oracle.stepping_sim(g, pol, par, exact=kw.get("exact", True), warmup=kw.get("warmup", False))
    assert st["rounds"] == len(tr_ref), (label, st["rounds"], len(tr_ref))
    for f in TRACE_FIELDS:
        if not np.array_equal(tr[f], tr_ref[f]):
            r = int(np.flatnonzero(tr[f] != tr_ref[f])[0])
            raise AssertionError(f"{label} round {r + 1} {f}: gpu {tr[f][r]} oracle {tr_ref[f][r]}")


@pytest.mark.parametrize("name", ["hub_chain", "grid256", "chain", "rmat12"])
def test_small_rounds_parity(cuda_device, name):
    import paper_2105_06145_b200 as P

    g = hub_chain() if name == "hub_chain" else (
        gen.chain(5000, np.random.default_rng(3).integers(1, 9, 4999).astype(np.uint32)) if name == "chain"
        else gen.make(name))
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g)
    saw_small = saw_grid = 0
    for pol, par, kw in POLICIES:
        for small in (True, False):
            got = P.dist_to_u64(h.run(g.source, pol, par, small=small, **kw))
            assert np.array_equal(got, want), (name, pol, par, small)
        # snapshot rounds: the trace with small rounds equals the oracle's simulation
        if kw.get("exact", True) and not (pol == "rho" and not kw):
            d, st, tr, _ = h.run(g.source, pol, par, trace_cap=1 << 16, snapshot=True, **kw)
            assert np.array_equal(P.dist_to_u64(d), want)
            _trace_same(g, tr, st, pol, par, kw, f"{name}/{pol}/{par}")
            saw_small += int(tr["small"].sum())
            saw_grid += int((tr["small"] == 0).sum())
            d0, st0, tr0, _ = h.run(g.source, pol, par, trace_cap=1 << 16, snapshot=True, small=False, **kw)
            assert tr0["small"].sum() == 0
            for f in TRACE_FIELDS:
                assert np.array_equal(tr[f], tr0[f]), (name, pol, par, f)
    assert saw_small > 0
    if name in ("hub_chain", "grid256", "rmat12"):
        assert saw_grid > 0  # the rounds were handed to the grid and back


def test_small_rounds_handoffs(cuda_device):
    """hub_chain under Bellman-Ford: small from round 1, the hub's round handed to the grid
    (too many arcs), the leaves' round on the grid (|Q| > 1024), small again on the tail."""
    import paper_2105_06145_b200 as P

    g = hub_chain()
    h = P.SSSP.from_graph(g)
    _, st, tr, _ = h.run(g.source, "bellman_ford", 0, trace_cap=1 << 16, snapshot=True)
    small = tr["small"].astype(bool)
    hub_round = int(np.flatnonzero(tr["edges"] >= 40000)[0])
    assert small[:hub_round].all()          # entered at round 1 and stayed
    assert not small[hub_round]             # frontier too large: undone and run by the grid
    assert not small[hub_round + 1]         # |Q| = 40000 leaves
    assert small[-1]                        # back to CTA 0 for the tail, and ended there
    assert st["rounds"] == oracle.k_n(g) + 1


def test_small_rounds_max_rounds(cuda_device):
    import paper_2105_06145_b200 as P

    g = gen.chain(3000, np.full(2999, 5, np.uint32))
    h = P.SSSP.from_graph(g)
    with pytest.raises(P.SSSPError) as e:
        h.run(g.source, "bellman_ford", 0, max_rounds=100)
    assert e.value.status == P.SSSP_ERR_ROUNDS
    # the handle stays usable
    want = oracle.dijkstra(g)
    assert np.array_equal(P.dist_to_u64(h.run(g.source, "bellman_ford", 0)), want)
