"""GPU parity for the standalone device LaB-PQ (sssp_pq_*), vs the naive PQ and selectors of oracle/."""
import numpy as np
import pytest

import oracle
from conftest import golden_value, load_golden

pytestmark = pytest.mark.gpu
INF = oracle.INF_INT
SPEC = load_golden("spec_examples.json")


def _P():
    import paper_2105_06145_b200 as P

    return P


def _keys(arr):
    import torch

    return torch.tensor(np.asarray(arr, dtype=np.uint64).view(np.int64), device="cuda")


@pytest.mark.parametrize("case", SPEC["pq"], ids=lambda c: c["name"])
def test_golden_pq(cuda_device, case):
    import torch

    P = _P()
    k = _keys(case["keys"])
    q = P.LabPQ(k)
    q.update(torch.tensor(case["updates"], dtype=torch.int32))
    out = q.extract(golden_value(case["theta"]))
    assert sorted(out.cpu().tolist()) == case["extracted"]
    assert sorted(q.queue().cpu().tolist()) == case["remaining"]
    assert q.size() == len(case["remaining"])


def test_lazy_update_semantics(cuda_device):
    """update, then lower the key, then extract with theta between -> extracted (keys read lazily)."""
    import torch

    P = _P()
    k = _keys([10, 10, 10])
    q = P.LabPQ(k)
    q.update(torch.tensor([0, 1], dtype=torch.int32))
    k[0] = 3
    assert q.extract(5).cpu().tolist() == [0]
    assert q.size() == 1


def test_pq_fuzz_vs_naive(cuda_device):
    """Random update batches (with duplicates), key decreases and extracts; sets must match."""
    import torch

    P = _P()
    rs = np.random.default_rng(2024)
    for trial in range(60):
        n = int(rs.integers(1, 513)) if trial < 50 else int(rs.integers(10000, 200000))
        keys_np = rs.integers(0, 1000, n).astype(np.uint64)
        k = _keys(keys_np)
        q = P.LabPQ(k)
        naive = oracle.NaivePQ(keys_np)
        for step in range(int(rs.integers(5, 30))):
            op = rs.integers(0, 3)
            if op == 0:
                ids = rs.integers(0, n, int(rs.integers(0, 2 * n + 1))).astype(np.int32)
                q.update(torch.from_numpy(ids))
                naive.update(ids)
            elif op == 1:
                sel = rs.integers(0, n, int(rs.integers(0, n + 1)))
                keys_np[sel] = np.minimum(keys_np[sel], rs.integers(0, 1000, len(sel)).astype(np.uint64))
                k.copy_(torch.from_numpy(keys_np.view(np.int64)).cuda())
            else:
                th = int(rs.integers(0, 1100)) if rs.random() < 0.9 else INF
                got = set(q.extract(th).cpu().tolist())
                want = naive.extract(th)
                assert got == want, (trial, step)
            assert q.size() == naive.size()
        assert set(q.queue().cpu().tolist()) == naive.ids


def test_extract_capacity_and_range_errors(cuda_device):
    import torch

    P = _P()
    k = _keys(np.arange(100))
    q = P.LabPQ(k)
    q.update(torch.arange(100, dtype=torch.int32))
    with pytest.raises(P.SSSPError) as e:
        q.extract(49, cap=10)
    assert e.value.status == P.SSSP_ERR_CAPACITY
    assert q.size() == 100  # unchanged
    assert sorted(q.extract(49, cap=50).cpu().tolist()) == list(range(50))
    q.update(torch.tensor([5, 100, -1], dtype=torch.int32))
    with pytest.raises(P.SSSPError) as e:
        q.size()
    assert e.value.status == P.SSSP_ERR_RANGE
    assert q.size() == 51  # the valid id was inserted, the error was reported once


def test_select_exact_and_sampled_parity(cuda_device):
    """Exact = k-th order statistic; sampled = the oracle's sampler replayed on the device queue order."""
    import torch

    P = _P()
    rs = np.random.default_rng(7)
    for t in range(25):
        n = int(rs.integers(2, 300000))
        keys_np = rs.integers(0, 1 << int(rs.integers(1, 50)), n).astype(np.uint64)
        k = _keys(keys_np)
        q = P.LabPQ(k)
        ids = np.unique(rs.integers(0, n, int(rs.integers(1, n + 1)))).astype(np.int32)
        q.update(torch.from_numpy(ids))
        order = q.queue().cpu().numpy()
        assert sorted(order.tolist()) == ids.tolist()
        qkeys = keys_np[order]
        for rho in {1, 2, max(1, len(ids) // 7), max(1, len(ids) - 1), len(ids), len(ids) + 5}:
            want = oracle.select_exact(qkeys, rho)
            assert q.select(rho, exact=True) == want
            for seed in (0, 99):
                assert q.select(rho, seed=seed) == oracle.select_sampled(qkeys, rho, seed=seed, round_=0)
        assert q.reduce_min() == int(qkeys.min())
    # full 64-bit keys: top bit set, SSSP_INF, heavy duplicates (all eight radix digits)
    for t in range(4):
        n = 50000
        pool = np.array([0, 1, 1 << 63, (1 << 64) - 1, (1 << 63) - 1, 12345], dtype=np.uint64)
        keys_np = np.where(rs.random(n) < 0.5, rs.choice(pool, n), rs.integers(0, 1 << 63, n, dtype=np.uint64) * 2 + 1)
        keys_np = keys_np.astype(np.uint64)
        q = P.LabPQ(_keys(keys_np))
        ids = np.unique(rs.integers(0, n, n)).astype(np.int32)
        q.update(torch.from_numpy(ids))
        qkeys = keys_np[q.queue().cpu().numpy()]
        for rho in (1, 7, len(ids) // 3, len(ids) // 2, len(ids) - 1):
            assert q.select(rho, exact=True) == oracle.select_exact(qkeys, rho), (t, rho)
    q = P.LabPQ(_keys([1, 2]))
    assert q.reduce_min() == INF and q.select(1) == INF
