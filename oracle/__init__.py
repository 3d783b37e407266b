"""ctypes wrapper over oracle/liboracle.so — the plain CPU reference.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_2105_06145_b200/) never imports it.  See oracle.h for the citations and
pins of every function.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
INF = np.uint64(0xFFFFFFFFFFFFFFFF)
INF_INT = 0xFFFFFFFFFFFFFFFF

RHO, DELTA, BF, DIJKSTRA, DELTA_STEPPING = 0, 1, 2, 3, 4
RHO_EXACT, RHO_WARMUP = 1, 2
POLICIES = {"rho": RHO, "delta": DELTA, "bellman_ford": BF, "dijkstra": DIJKSTRA, "delta_stepping": DELTA_STEPPING}

ROUND_DTYPE = np.dtype([("qsize", "<i8"), ("fsize", "<i8"), ("edges", "<i8"), ("inserts", "<i8"),
                        ("succ", "<i8"), ("theta", "<u8"), ("pad0", "<i8"), ("pad1", "<i8")])


def build(verbose: bool = False) -> str:
    import subprocess

    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, os.path.join(_HERE, "oracle.c")]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    srcs = [os.path.join(_HERE, f) for f in ("oracle.c", "oracle.h")]
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(s) for s in srcs):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    lib.oracle_dijkstra.restype = i64
    lib.oracle_dijkstra.argtypes = [i32, vp, vp, vp, i32, vp, vp]
    lib.oracle_dijkstra_budget.restype = i64
    lib.oracle_dijkstra_budget.argtypes = [i32, vp, vp, vp, i32, vp, i64, vp]
    lib.oracle_bellman_ford.restype = i64
    lib.oracle_bellman_ford.argtypes = [i32, vp, vp, vp, i32, vp]
    lib.oracle_bfs.restype = i64
    lib.oracle_bfs.argtypes = [i32, vp, vp, i32, vp]
    lib.oracle_certify.restype = ctypes.c_int
    lib.oracle_certify.argtypes = [i32, vp, vp, vp, i32, vp, vp]
    lib.oracle_stepping_sim.restype = i64
    lib.oracle_stepping_sim.argtypes = [i32, vp, vp, vp, i32, ctypes.c_int, u64, ctypes.c_uint32, u64, i64, vp, vp,
                                        i64, vp]
    lib.oracle_select_sampled.restype = u64
    lib.oracle_select_sampled.argtypes = [vp, i64, u64, u64, u64]
    lib.oracle_select_exact.restype = u64
    lib.oracle_select_exact.argtypes = [vp, i64, u64]
    _lib = lib
    return lib


def _csr(g):
    off = np.ascontiguousarray(g.offsets, dtype=np.int32)
    idx = np.ascontiguousarray(g.indices, dtype=np.int32)
    w = np.ascontiguousarray(g.weights, dtype=np.uint32)
    if len(idx) == 0:  # keep valid pointers for m = 0
        idx = np.zeros(1, np.int32)
        w = np.zeros(1, np.uint32)
    return off, idx, w


def dijkstra(g, source=None, with_hops=False):
    """Exact distances (uint64, INF = 2^64-1); with_hops also returns min-hop counts."""
    s = g.source if source is None else source
    off, idx, w = _csr(g)
    dist = np.empty(g.n, np.uint64)
    hops = np.empty(g.n, np.int32) if with_hops else None
    _load().oracle_dijkstra(g.n, off.ctypes.data, idx.ctypes.data, w.ctypes.data, s, dist.ctypes.data,
                            hops.ctypes.data if with_hops else None)
    return (dist, hops) if with_hops else dist


def dijkstra_budget(g, source, arc_budget, return_dist=False):
    """Dijkstra stopped before the first pop once `arc_budget` arcs were scanned (the measurement
    sample of bench.py); returns (arcs_scanned, settled) [, tentative distances]."""
    off, idx, w = _csr(g)
    dist = np.empty(g.n, np.uint64)
    settled = ctypes.c_int64(0)
    scanned = _load().oracle_dijkstra_budget(g.n, off.ctypes.data, idx.ctypes.data, w.ctypes.data, source,
                                             dist.ctypes.data, int(arc_budget), ctypes.addressof(settled))
    if return_dist:
        return int(scanned), int(settled.value), dist
    return int(scanned), int(settled.value)


def k_n(g, source=None):
    """Shortest-path-tree depth in hops."""
    _, hops = dijkstra(g, source, with_hops=True)
    return int(hops.max()) if (hops >= 0).any() else 0


def bellman_ford(g, source=None):
    s = g.source if source is None else source
    off, idx, w = _csr(g)
    dist = np.empty(g.n, np.uint64)
    passes = _load().oracle_bellman_ford(g.n, off.ctypes.data, idx.ctypes.data, w.ctypes.data, s, dist.ctypes.data)
    return dist, int(passes)


def bfs(g, source=None):
    s = g.source if source is None else source
    off, idx, _ = _csr(g)
    lvl = np.empty(g.n, np.int32)
    _load().oracle_bfs(g.n, off.ctypes.data, idx.ctypes.data, s, lvl.ctypes.data)
    return lvl


def certify(g, dist, source=None):
    """0 if dist is the exact SSSP solution (certificate (i)-(iv)), else (condition, vertex)."""
    s = g.source if source is None else source
    off, idx, w = _csr(g)
    d = np.ascontiguousarray(dist, dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_certify(g.n, off.ctypes.data, idx.ctypes.data, w.ctypes.data, s, d.ctypes.data,
                                ctypes.addressof(bad))
    return 0 if rc == 0 else (int(rc), int(bad.value))


def stepping_sim(g, policy, param=0, source=None, exact=True, warmup=False, seed=0, max_rounds=10**8,
                 trace_cap=1 << 20, ext_counts=False):
    """Alg. 1 simulated with snapshot semantics; returns (dist, trace[rounds], ext_count|None)."""
    s = g.source if source is None else source
    pol = POLICIES[policy] if isinstance(policy, str) else policy
    off, idx, w = _csr(g)
    dist = np.empty(g.n, np.uint64)
    trace = np.zeros(trace_cap, ROUND_DTYPE)
    ext = np.empty(g.n, np.int32) if ext_counts else None
    flags = (RHO_EXACT if exact else 0) | (RHO_WARMUP if warmup else 0)
    rounds = _load().oracle_stepping_sim(g.n, off.ctypes.data, idx.ctypes.data, w.ctypes.data, s, pol, int(param),
                                         flags, int(seed), int(max_rounds), dist.ctypes.data, trace.ctypes.data,
                                         trace_cap, ext.ctypes.data if ext_counts else None)
    if rounds < 0:
        raise RuntimeError("stepping_sim exceeded max_rounds")
    return dist, trace[: min(rounds, trace_cap)], ext


def select_sampled(keys, rho, seed=0, round_=0):
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    if len(k) == 0:
        return INF_INT
    return int(_load().oracle_select_sampled(k.ctypes.data, len(k), int(rho), int(seed), int(round_)))


def select_exact(keys, rho):
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    if len(k) == 0:
        return INF_INT
    return int(_load().oracle_select_exact(k.ctypes.data, len(k), int(rho)))


class NaivePQ:
    """Naive LaB-PQ (Table tab:interface): a set of ids over a key map.

    Update(id) inserts or notifies; Extract(theta) returns and removes every id with
    key <= theta.  Used to pin the device PQ (extract compared as sets).
    """

    def __init__(self, keys: np.ndarray):
        self.keys = keys  # the mapping function delta, read at Extract time
        self.ids: set[int] = set()

    def update(self, ids):
        self.ids.update(int(i) for i in ids)

    def extract(self, theta):
        out = {i for i in self.ids if int(self.keys[i]) <= int(theta)}
        self.ids -= out
        return out

    def size(self):
        return len(self.ids)
