#!/usr/bin/env python
"""Per-round floor of the round loop: a path graph makes one vertex per round (exploration, not the bench)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

n = int(os.environ.get("FLOOR_N", "20000"))
g = gen.chain(n, np.ones(n - 1, np.uint32))
h = P.SSSP.from_graph(g)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
for pol, par in (("bellman_ford", 0), ("rho", 1 << 12), ("delta", 1)):
    for snap in (False, True):
        for _ in range(2):
            h.run(0, pol, par, out=d, snapshot=snap)
        ks = []
        for _ in range(3):
            h.run(0, pol, par, out=d, snapshot=snap)
            ks.append(h.last_stats["kernel_ms"])
        rounds = h.last_stats["rounds"]
        _, st, tr, _ = h.run(0, pol, par, out=d, snapshot=snap, trace_cap=1 << 16)
        med = {k: statistics.median(tr[k].tolist()) / 1e3 for k in ("t_theta_ns", "t_extract_ns", "t_relax_ns")}
        print(f"{pol:13s} snap={snap!s:5s} rounds {rounds}  {statistics.median(ks) * 1e3 / rounds:6.2f} us/round  "
              f"grid {st['grid_blocks']}x{st['block_threads']}  stats-run medians (us): {med}", flush=True)
