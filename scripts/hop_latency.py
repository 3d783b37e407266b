#!/usr/bin/env python
"""Fusion hop latency: on a path graph with Delta* large, each round is one fusion chain of
`fuse_budget` hops (one vertex per batch), so time/round = overhead + budget * hop.  Two
budgets give both terms (exploration, not the bench)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

n = 1 << 17
for name, g in (("path", gen.chain(n, np.full(n - 1, 5, np.uint32))),):
    h = P.SSSP.from_graph(g)
    d = torch.empty(g.n, dtype=torch.int64, device="cuda")
    res = {}
    for fb in (16, 32, 64, 128):
        ts = []
        for r in range(3):
            h.run(g.source, "delta", 1 << 40, out=d, fuse_budget=fb)
            ts.append(h.last_stats["kernel_ms"])
        ms = statistics.median(ts)
        rounds = h.last_stats["rounds"]
        res[fb] = (ms, rounds)
        print(f"{name} budget {fb:4d}: {ms:8.3f} ms, {rounds} rounds, {ms * 1e3 / rounds:7.2f} us/round", flush=True)
    a, b = res[32], res[128]
    # us/round = ovh + fb * hop
    hop = (b[0] * 1e3 / b[1] - a[0] * 1e3 / a[1]) / (128 - 32)
    ovh = a[0] * 1e3 / a[1] - 32 * hop
    print(f"{name}: hop latency {hop:.2f} us, per-round overhead {ovh:.2f} us")
