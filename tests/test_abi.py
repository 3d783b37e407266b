"""CPU-side checks of the C-ABI library: it loads and exports every symbol include/sssp.h declares.

No compute calls (there is no GPU here); only pure host queries are exercised.
"""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sssp.h")
LIB = os.path.join(ROOT, "paper_2105_06145_b200", "libsssp.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sssp_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("sssp_workspace_bytes", "sssp_create", "sssp_run", "sssp_run_ex", "sssp_run_host", "sssp_destroy",
              "sssp_pq_create", "sssp_pq_update", "sssp_pq_extract", "sssp_pq_size", "sssp_pq_select",
              "sssp_pq_reduce_min", "sssp_pq_destroy", "sssp_status_string", "sssp_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libsssp.so not built (run __graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sssp_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_binding_loads_and_mirrors_names():
    import paper_2105_06145_b200 as P

    assert P.sssp_abi_version() == 1
    assert set(declared_functions()) == set(P.EXPORTED_SYMBOLS)
    assert P.sssp_status_string(P.SSSP_ERR_RANGE) == b"SSSP_ERR_RANGE"


def test_workspace_sizing_host_only():
    import paper_2105_06145_b200 as P

    assert P.sssp_workspace_bytes(0, 0, 0) == 0
    assert P.sssp_workspace_bytes(-5, 0, 0) == 0
    assert P.sssp_workspace_bytes(10, -1, 0) == 0
    assert P.sssp_workspace_bytes(10, 1 << 31, 0) == 0
    small = P.sssp_workspace_bytes(1, 0, 0)
    assert small > 0
    n, m = 1 << 24, 520_000_000
    big = P.sssp_workspace_bytes(n, m, 0)
    # interleaved arcs 8m; dist x2 16n + two sharded queues (3n ids each) 24n + light
    # frontier 16n = 56n; chunk descriptors: 3 x 16 B x (m/chunk + m/(light+1)) with
    # chunk >= 128 arcs and light >= 32 (sharded at 2x + spill); counters/samples < 64 MiB
    # isolated-vertex compaction (m >= 20 n): offsets 4n + two id maps 8n + distances 8n
    relabel = 20 * n
    assert 8 * m + 56 * n + relabel < big < 8 * m + 56 * n + relabel + 48 * (m // 128 + m // 33 + 1) + (64 << 20)
    assert abs(P.sssp_workspace_bytes(n, m, P.SSSP_NO_RELABEL) - (big - relabel)) < 4096  # alignment slack
    assert P.sssp_pq_workspace_bytes(1000) > 8 * 1000 // 8


def test_create_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call."""
    import ctypes

    import paper_2105_06145_b200 as P

    h = ctypes.c_void_p(0)
    z = ctypes.c_void_p(0)
    assert P.sssp_create(0, 0, z, z, z, z, 0, z, 0, ctypes.byref(h)) == P.SSSP_ERR_INVALID
    assert b"n=0" in P.sssp_last_error()
    assert P.sssp_create(5, 4, z, z, z, z, 0, z, 0, ctypes.byref(h)) == P.SSSP_ERR_INVALID
    assert P.sssp_run(None, 0, 0, 1, z, None) == P.SSSP_ERR_INVALID
    assert P.sssp_pq_create(10, z, z, 0, z, ctypes.byref(h)) == P.SSSP_ERR_INVALID


def test_product_does_not_import_oracle():
    """The CUDA path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_2105_06145_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "sssp.h" not in src and "paper_2105_06145_b200" not in src
