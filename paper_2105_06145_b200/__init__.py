"""B200-native stepping SSSP (arXiv 2105.06145) — thin Python binding over libsssp.so.

Every step of the hot path runs in the CUDA kernels behind the C ABI declared in
include/sssp.h; this module only marshals arguments (torch tensors -> device
pointers, the current torch stream -> cudaStream_t).  There is no CPU fallback:
importing fails loudly when the extension is missing, and calls fail loudly
without a CUDA device.

Low-level names mirror the C ABI (sssp_create, sssp_run, sssp_pq_update, ...);
`SSSP` and `LabPQ` are small convenience wrappers over them.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SSSP_LIB selects an in-tree tuning variant built by build.py --out (same ABI)
LIB_PATH = os.environ.get("SSSP_LIB") or os.path.join(_HERE, "libsssp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

INF = 0xFFFFFFFFFFFFFFFF
SSSP_OK, SSSP_ERR_INVALID, SSSP_ERR_INVALID_GRAPH, SSSP_ERR_RANGE = 0, -1, -2, -3
SSSP_ERR_CAPACITY, SSSP_ERR_CUDA, SSSP_ERR_ROUNDS, SSSP_ERR_DEVICE, SSSP_ERR_INTERNAL = -4, -5, -6, -7, -8
SSSP_RHO, SSSP_DELTA, SSSP_BELLMAN_FORD, SSSP_DIJKSTRA, SSSP_DELTA_STEPPING = 0, 1, 2, 3, 4
POLICIES = {"rho": SSSP_RHO, "delta": SSSP_DELTA, "bellman_ford": SSSP_BELLMAN_FORD, "bf": SSSP_BELLMAN_FORD,
            "dijkstra": SSSP_DIJKSTRA, "delta_stepping": SSSP_DELTA_STEPPING}
SSSP_VALIDATE = 1
SSSP_NO_RELABEL = 2
SSSP_RUN_RHO_EXACT, SSSP_RUN_NO_WARMUP, SSSP_RUN_STATS, SSSP_RUN_SNAPSHOT, SSSP_RUN_NO_NEARFAR = 1, 2, 4, 8, 16
SSSP_RUN_NO_FUSE, SSSP_RUN_BIDIR, SSSP_RUN_NO_SMALL = 32, 64, 128
SSSP_SELECT_SAMPLED, SSSP_SELECT_EXACT = 0, 1


class SSSPError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.sssp_status_string(status).decode()
        detail = _lib.sssp_last_error().decode()
        super().__init__(f"{where}: {msg}: {detail}")


class sssp_run_opts(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_uint32), ("fuse_budget", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("max_rounds", ctypes.c_int64), ("d_trace", ctypes.c_void_p), ("trace_cap", ctypes.c_int64),
                ("d_ext_count", ctypes.c_void_p), ("fuse_depth", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class sssp_run_stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("extracted", ctypes.c_int64), ("edges", ctypes.c_int64),
                ("succ", ctypes.c_int64), ("inserts", ctypes.c_int64), ("queue_scanned", ctypes.c_int64),
                ("max_queue", ctypes.c_int64), ("max_frontier", ctypes.c_int64), ("dense_scanned", ctypes.c_int64),
                ("grid_blocks", ctypes.c_int32),
                ("block_threads", ctypes.c_int32), ("kernel_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: (float if k == "kernel_ms" else int)(getattr(self, k)) for k, _ in self._fields_}


ROUND_FIELDS = ["qsize", "fsize", "edges", "inserts", "succ", "theta", "nheavy", "t_theta_ns", "t_extract_ns",
                "t_relax_ns", "qnear", "dense", "busy_a_ns", "busy_b_ns",
                "busy_a_max_ns", "fused", "t_near_ns", "prof_scan", "prof_take", "prof_relax", "prof_flush",
                "prof_fuse", "prof_fuse_batches", "prof_steps", "prof_step_cyc", "small"]
ROUND_WORDS = len(ROUND_FIELDS)

_vp, _i32, _i64, _u64, _u32, _sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_uint32, ctypes.c_size_t)
_st = ctypes.c_int
_sigs = {
    "sssp_workspace_bytes": (_sz, [_i32, _i64, _u32]),
    "sssp_create": (_st, [_i32, _i64, _vp, _vp, _vp, _vp, _sz, _vp, _u32, ctypes.POINTER(_vp)]),
    "sssp_run": (_st, [_vp, _i32, ctypes.c_int, _u64, _vp, ctypes.POINTER(sssp_run_stats)]),
    "sssp_run_ex": (_st, [_vp, _i32, ctypes.c_int, _u64, ctypes.POINTER(sssp_run_opts), _vp,
                          ctypes.POINTER(sssp_run_stats)]),
    "sssp_run_host": (_st, [_vp, _i32, ctypes.c_int, _u64, _vp, ctypes.POINTER(sssp_run_stats)]),
    "sssp_run_batch_host": (_st, [_vp, _vp, _i32, ctypes.c_int, _u64, ctypes.POINTER(sssp_run_opts), _vp,
                                  ctypes.POINTER(sssp_run_stats)]),
    "sssp_destroy": (_st, [_vp]),
    "sssp_pq_workspace_bytes": (_sz, [_i32]),
    "sssp_pq_create": (_st, [_i32, _vp, _vp, _sz, _vp, ctypes.POINTER(_vp)]),
    "sssp_pq_update": (_st, [_vp, _vp, _i64]),
    "sssp_pq_extract": (_st, [_vp, _u64, _vp, _i64, ctypes.POINTER(_i64)]),
    "sssp_pq_size": (_st, [_vp, ctypes.POINTER(_i64)]),
    "sssp_pq_select": (_st, [_vp, _u64, _u64, _u32, ctypes.POINTER(_u64)]),
    "sssp_pq_reduce_min": (_st, [_vp, ctypes.POINTER(_u64)]),
    "sssp_pq_queue": (_st, [_vp, _vp, _i64, ctypes.POINTER(_i64)]),
    "sssp_pq_destroy": (_st, [_vp]),
    "sssp_status_string": (ctypes.c_char_p, [_st]),
    "sssp_last_error": (ctypes.c_char_p, []),
    "sssp_abi_version": (_i32, []),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f  # the C names, unchanged

EXPORTED_SYMBOLS = sorted(_sigs)


def _check(status, where):
    if status != SSSP_OK:
        raise SSSPError(status, where)


def _torch():
    import torch

    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else ctypes.c_void_p(0)


class SSSP:
    """Handle over a device-resident CSR (int32 offsets/indices, uint32 weights as int32 or uint32 tensors)."""

    def __init__(self, offsets, indices, weights, validate: bool = False, stream=None, relabel: bool = True):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("SSSP needs a CUDA device (no CPU fallback)")
        dev = offsets.device
        assert dev.type == "cuda" and indices.device == dev and weights.device == dev
        assert offsets.dtype == torch.int32 and indices.dtype == torch.int32
        assert weights.dtype in (torch.int32, torch.uint32)
        self.n = offsets.numel() - 1
        self.m = indices.numel()
        self.offsets, self.indices, self.weights = offsets, indices, weights  # keep borrowed buffers alive
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        flags = (SSSP_VALIDATE if validate else 0) | (0 if relabel else SSSP_NO_RELABEL)
        nbytes = sssp_workspace_bytes(self.n, self.m, flags)
        if nbytes == 0:
            raise ValueError(f"graph size out of range (n={self.n}, m={self.m})")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        base = self.workspace.data_ptr()
        self._ws_ptr = (base + 255) // 256 * 256
        h = ctypes.c_void_p(0)
        _check(sssp_create(self.n, self.m, _ptr(offsets), _ptr(indices), _ptr(weights), ctypes.c_void_p(self._ws_ptr),
                           nbytes, _stream_ptr(self.stream), flags, ctypes.byref(h)), "sssp_create")
        self._h = h

    @staticmethod
    def from_graph(g, device="cuda", validate=False, relabel=True):
        """Upload a host CSR (gen.Graph or anything with offsets/indices/weights numpy arrays)."""
        torch = _torch()
        off = torch.from_numpy(g.offsets).to(device)
        idx = torch.from_numpy(g.indices).to(device)
        w = torch.from_numpy(g.weights.view("int32")).to(device)
        return SSSP(off, idx, w, validate=validate, relabel=relabel)

    def run(self, source, policy="rho", param=0, out=None, stats=False, trace_cap=0, ext_counts=False,
            exact=False, warmup=True, seed=0, max_rounds=0, snapshot=False, nearfar=True, fuse=True,
            fuse_budget=0, bidir=False, fuse_depth=0, small=True):
        """Alg. 1 from `source`; returns a uint64-valued int64 tensor of distances (INF = -1 as int64).

        With stats=True returns (dist, stats_dict, trace ndarray | None, ext_count tensor | None)."""
        torch = _torch()
        pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
        dev = self.offsets.device
        if out is None:
            out = torch.empty(self.n, dtype=torch.int64, device=dev)
        # the kernel writes n uint64 words through the raw pointer: refuse anything smaller
        if not (out.device == dev and out.dtype in (torch.int64, torch.uint64) and out.is_contiguous()
                and out.numel() >= self.n):
            raise ValueError(f"out must be a contiguous int64/uint64 tensor of >= {self.n} elements on {dev} "
                             f"(got {tuple(out.shape)} {out.dtype} on {out.device})")
        o = sssp_run_opts()
        o.flags = (SSSP_RUN_RHO_EXACT if exact else 0) | (0 if warmup else SSSP_RUN_NO_WARMUP) | \
                  (SSSP_RUN_STATS if (stats or trace_cap) else 0) | (SSSP_RUN_SNAPSHOT if snapshot else 0) | \
                  (0 if nearfar else SSSP_RUN_NO_NEARFAR) | (0 if fuse else SSSP_RUN_NO_FUSE) | \
            (SSSP_RUN_BIDIR if bidir else 0) | (0 if small else SSSP_RUN_NO_SMALL)
        o.fuse_budget = fuse_budget
        o.fuse_depth = fuse_depth
        o.seed = seed
        o.max_rounds = max_rounds
        trace = None
        ext = None
        with torch.cuda.stream(self.stream):  # the fills are ordered before the launch on the same stream
            if trace_cap:
                trace = torch.zeros(trace_cap * ROUND_WORDS, dtype=torch.int64, device=dev)
                o.d_trace = trace.data_ptr()
                o.trace_cap = trace_cap
            if ext_counts:
                ext = torch.zeros(self.n, dtype=torch.int32, device=dev)
                o.d_ext_count = ext.data_ptr()
        st = sssp_run_stats()
        with torch.cuda.stream(self.stream):
            _check(sssp_run_ex(self._h, int(source), pol, int(param), ctypes.byref(o), _ptr(out), ctypes.byref(st)),
                   "sssp_run")
        self.last_stats = st.as_dict()
        if not (stats or trace_cap or ext_counts):
            return out
        tr = None
        if trace is not None:
            import numpy as np

            r = min(int(st.rounds), trace_cap)
            raw = trace.view(-1, ROUND_WORDS)[:r].cpu().numpy()
            tr = np.zeros(r, dtype=[(f, "<u8" if f == "theta" else "<i8") for f in ROUND_FIELDS])
            for i, f in enumerate(ROUND_FIELDS):
                tr[f] = raw[:, i].view("<u8") if f == "theta" else raw[:, i]
        return out, st.as_dict(), tr, ext

    def run_host(self, source, policy="rho", param=0, out_host=None):
        """End-to-end call: distances land in host memory (pinned tensor recommended)."""
        torch = _torch()
        pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
        if out_host is None:
            out_host = torch.empty(self.n, dtype=torch.int64, pin_memory=True)
        st = sssp_run_stats()
        _check(sssp_run_host(self._h, int(source), pol, int(param), ctypes.c_void_p(out_host.data_ptr()),
                             ctypes.byref(st)), "sssp_run_host")
        self.last_stats = st.as_dict()
        return out_host

    def run_batch_host(self, sources, policy="rho", param=0, out_host=None, seed=0):
        """End-to-end multi-source call: k sources, k x n distances in host memory (pinned
        tensor recommended); the read-back of one source overlaps the next run."""
        import numpy as np

        torch = _torch()
        pol = POLICIES[policy] if isinstance(policy, str) else int(policy)
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int32))
        k = len(src)
        if out_host is None:
            out_host = torch.empty((k, self.n), dtype=torch.int64, pin_memory=True)
        o = sssp_run_opts()
        o.seed = seed
        st = sssp_run_stats()
        _check(sssp_run_batch_host(self._h, ctypes.c_void_p(src.ctypes.data), k, pol, int(param), ctypes.byref(o),
                                   ctypes.c_void_p(out_host.data_ptr()), ctypes.byref(st)), "sssp_run_batch_host")
        self.last_stats = st.as_dict()
        return out_host

    def close(self):
        if getattr(self, "_h", None):
            sssp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LabPQ:
    """Device LaB-PQ over ids [0, n) keyed by a borrowed int64/uint64 device tensor."""

    def __init__(self, keys, stream=None):
        torch = _torch()
        assert keys.device.type == "cuda" and keys.dtype in (torch.int64, torch.uint64)
        self.keys = keys
        self.n = keys.numel()
        self.stream = stream if stream is not None else torch.cuda.current_stream(keys.device)
        nbytes = sssp_pq_workspace_bytes(self.n)
        if nbytes == 0:
            raise ValueError(f"n={self.n} out of range")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=keys.device)
        ws = (self.workspace.data_ptr() + 255) // 256 * 256
        q = ctypes.c_void_p(0)
        _check(sssp_pq_create(self.n, _ptr(keys), ctypes.c_void_p(ws), nbytes, _stream_ptr(self.stream),
                              ctypes.byref(q)), "sssp_pq_create")
        self._q = q

    def update(self, ids):
        torch = _torch()
        ids = ids.to(device=self.keys.device, dtype=torch.int32).contiguous()
        self._last_ids = ids  # keep alive until the stream consumes it
        _check(sssp_pq_update(self._q, _ptr(ids), ids.numel()), "sssp_pq_update")

    def extract(self, theta, cap=None, out=None):
        torch = _torch()
        cap = self.n if cap is None else cap
        if out is None:
            out = torch.empty(max(cap, 1), dtype=torch.int32, device=self.keys.device)
        elif not (out.device == self.keys.device and out.dtype == torch.int32 and out.is_contiguous()
                  and out.numel() >= max(cap, 1)):
            raise ValueError(f"out must be a contiguous int32 tensor of >= {max(cap, 1)} elements on {self.keys.device}")
        cnt = ctypes.c_int64(0)
        _check(sssp_pq_extract(self._q, int(theta), _ptr(out), cap, ctypes.byref(cnt)), "sssp_pq_extract")
        return out[: cnt.value]

    def size(self):
        s = ctypes.c_int64(0)
        _check(sssp_pq_size(self._q, ctypes.byref(s)), "sssp_pq_size")
        return int(s.value)

    def select(self, rho, seed=0, exact=False):
        t = ctypes.c_uint64(0)
        _check(sssp_pq_select(self._q, int(rho), int(seed), SSSP_SELECT_EXACT if exact else SSSP_SELECT_SAMPLED,
                              ctypes.byref(t)), "sssp_pq_select")
        return int(t.value)

    def reduce_min(self):
        t = ctypes.c_uint64(0)
        _check(sssp_pq_reduce_min(self._q, ctypes.byref(t)), "sssp_pq_reduce_min")
        return int(t.value)

    def queue(self, out=None):
        torch = _torch()
        if out is None:
            out = torch.empty(max(self.n, 1), dtype=torch.int32, device=self.keys.device)
        elif not (out.device == self.keys.device and out.dtype == torch.int32 and out.is_contiguous()
                  and out.numel() >= max(self.n, 1)):
            raise ValueError(f"out must be a contiguous int32 tensor of >= {max(self.n, 1)} elements on {self.keys.device}")
        cnt = ctypes.c_int64(0)
        _check(sssp_pq_queue(self._q, _ptr(out), self.n, ctypes.byref(cnt)), "sssp_pq_queue")
        return out[: cnt.value]

    def close(self):
        if getattr(self, "_q", None):
            sssp_pq_destroy(self._q)
            self._q = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_to_u64(t):
    """int64 tensor of distances -> numpy uint64 (INF = 2^64-1)."""
    return t.cpu().numpy().view("uint64")
