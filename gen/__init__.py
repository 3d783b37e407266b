"""Seeded synthetic graph inputs (CSR) shared by the oracle side and the CUDA side.

This module is input plumbing only: it holds none of the SSSP method's arithmetic.
The five workload recipes stand in for the paper's graphs (PAPER.md P:1527-1528,
P:1598: social/web graphs with weights uniform in [1,2^18), road graphs with deep
shortest-path trees); see DESIGN.md "Inputs" and SURVEY.md §8(d).

Every random value is a counter-based splitmix64 hash of (seed, key), so outputs
are bit-identical for any thread count.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgen.so")

W_UNIFORM, W_LOGUNIFORM, W_CONST = 0, 1, 2


class _GenGraph(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("m", ctypes.c_int64),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("indices", ctypes.POINTER(ctypes.c_int32)),
        ("weights", ctypes.POINTER(ctypes.c_uint32)),
        ("xy", ctypes.POINTER(ctypes.c_double)),
    ]


def build(verbose: bool = False) -> str:
    import subprocess

    src = os.path.join(_HERE, "gen.c")
    cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-o", _LIB_PATH, src, "-lm"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "gen.c")):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.POINTER(_GenGraph)
    lib.gen_grid.restype = P
    lib.gen_grid.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32]
    lib.gen_rmat.restype = P
    lib.gen_rmat.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                             ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32]
    lib.gen_random.restype = P
    lib.gen_random.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                               ctypes.c_uint32]
    lib.gen_rgg_knn.restype = P
    lib.gen_rgg_knn.argtypes = [ctypes.c_int32, ctypes.c_int, ctypes.c_uint64]
    lib.gen_from_arcs.restype = P
    lib.gen_from_arcs.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int]
    lib.gen_free.restype = None
    lib.gen_free.argtypes = [P]
    lib.gen_num_threads.restype = ctypes.c_int
    _lib = lib
    return lib


@dataclass
class Graph:
    """Host CSR: int32 offsets[n+1], int32 indices[m], uint32 weights[m]."""

    n: int
    m: int
    offsets: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    source: int = 0
    name: str = ""
    xy: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    @property
    def max_weight(self) -> int:
        return int(self.weights.max()) if self.m else 0


def _take(ptr, name="") -> Graph:
    if not ptr:
        raise ValueError(f"generator {name} failed (bad parameters or out of memory)")
    lib = _load()
    g = ptr.contents
    n, m = int(g.n), int(g.m)
    off = np.ctypeslib.as_array(g.offsets, shape=(n + 1,)).copy()
    idx = np.ctypeslib.as_array(g.indices, shape=(max(m, 1),))[:m].copy()
    w = np.ctypeslib.as_array(g.weights, shape=(max(m, 1),))[:m].copy()
    xy = np.ctypeslib.as_array(g.xy, shape=(2 * n,)).copy().reshape(n, 2) if g.xy else None
    lib.gen_free(ptr)
    return Graph(n=n, m=m, offsets=off, indices=idx, weights=w, xy=xy, name=name)


def max_degree_vertex(g: Graph) -> int:
    """Highest-degree vertex, lowest id among ties (reading R13)."""
    return int(np.argmax(g.degrees)) if g.n else 0


def grid(rows: int, cols: int, seed: int, wmax: int = 65535, const_weight: int | None = None) -> Graph:
    """4-neighbour grid, id = r*cols + c, one weight per undirected edge in [1, wmax]."""
    if const_weight is not None:
        g = _take(_load().gen_grid(rows, cols, seed, W_CONST, const_weight), f"grid{rows}x{cols}")
    else:
        g = _take(_load().gen_grid(rows, cols, seed, W_UNIFORM, wmax), f"grid{rows}x{cols}")
    g.source = 0
    return g


def rmat(scale: int, seed: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, weights: str = "uniform18") -> Graph:
    """R-MAT, symmetrised, self-loops dropped, deduplicated; source = max-degree vertex."""
    if weights == "uniform18":
        wm, wp = W_UNIFORM, (1 << 18) - 1  # [1, 2^18)
    elif weights == "log20":
        wm, wp = W_LOGUNIFORM, 20  # floor(2^(20u)) in [1, 2^20)
    else:
        raise ValueError(weights)
    g = _take(_load().gen_rmat(scale, edge_factor, a, b, c, seed, wm, wp), f"rmat{scale}")
    g.source = max_degree_vertex(g)
    return g


def rgg_knn(n: int, seed: int, k: int = 4) -> Graph:
    """Random geometric kNN graph in the unit square; source = point nearest (0.5, 0.5)."""
    g = _take(_load().gen_rgg_knn(n, k, seed), f"rgg{n}")
    d2 = (g.xy[:, 0] - 0.5) ** 2 + (g.xy[:, 1] - 0.5) ** 2
    g.source = int(np.argmin(d2))  # argmin returns the lowest id among ties
    return g


def random_graph(n: int, draws: int, seed: int, directed: bool = False, wmax: int = (1 << 18) - 1) -> Graph:
    """G(n, draws) with hashed endpoints, weights uniform in [1, wmax]."""
    g = _take(_load().gen_random(n, draws, int(directed), seed, W_UNIFORM, wmax), f"random{n}")
    g.source = 0
    return g


def from_arcs(n: int, src, dst, w, symmetrise: bool = False, source: int = 0, name: str = "arcs") -> Graph:
    """CSR from explicit arcs; duplicate arcs keep the minimum weight; rows sorted by target."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.uint32)
    assert len(src) == len(dst) == len(w)
    if len(src):
        assert src.min() >= 0 and src.max() < n and dst.min() >= 0 and dst.max() < n
    g = _take(_load().gen_from_arcs(n, len(src), src.ctypes.data, dst.ctypes.data, w.ctypes.data, int(symmetrise)),
              name)
    g.source = source
    return g


def chain(n: int, weights=None, source: int = 0) -> Graph:
    w = np.ones(n - 1, dtype=np.uint32) if weights is None else np.asarray(weights, dtype=np.uint32)
    s = np.arange(n - 1)
    return from_arcs(n, s, s + 1, w, symmetrise=True, source=source, name=f"chain{n}")


def star(leaves: int, weights=None) -> Graph:
    w = np.ones(leaves, dtype=np.uint32) if weights is None else np.asarray(weights, dtype=np.uint32)
    return from_arcs(leaves + 1, np.zeros(leaves), np.arange(1, leaves + 1), w, symmetrise=True, source=0,
                     name=f"star{leaves}")


# ---------------------------------------------------------------------------------------------
# The five BASELINE.json configurations; seeds 1..5.
# ---------------------------------------------------------------------------------------------
CONFIGS = {
    "grid256": dict(kind="grid", rows=256, cols=256, seed=1),
    "rmat20": dict(kind="rmat", scale=20, seed=2, weights="uniform18"),
    "rgg4m": dict(kind="rgg", n=1 << 22, seed=3),
    "rmat24": dict(kind="rmat", scale=24, seed=4, weights="log20"),
    "grid4096": dict(kind="grid", rows=4096, cols=4096, seed=5),
    # reduced-size siblings used by CPU tests and quick GPU parity cases
    "grid64": dict(kind="grid", rows=64, cols=64, seed=1),
    "rmat12": dict(kind="rmat", scale=12, seed=2, weights="uniform18"),
    "rmat14log": dict(kind="rmat", scale=14, seed=4, weights="log20"),
    "rgg64k": dict(kind="rgg", n=1 << 16, seed=3),
    "grid1024": dict(kind="grid", rows=1024, cols=1024, seed=5),
    "rgg1m": dict(kind="rgg", n=1 << 20, seed=3),
}

FULL_CONFIGS = ["grid256", "rmat20", "rgg4m", "rmat24", "grid4096"]


def make(name: str) -> Graph:
    c = dict(CONFIGS[name])
    kind = c.pop("kind")
    if kind == "grid":
        g = grid(c["rows"], c["cols"], c["seed"])
    elif kind == "rmat":
        g = rmat(c["scale"], c["seed"], weights=c["weights"])
    elif kind == "rgg":
        g = rgg_knn(c["n"], c["seed"])
    else:
        raise ValueError(kind)
    g.name = name
    return g


def num_threads() -> int:
    return int(_load().gen_num_threads())
