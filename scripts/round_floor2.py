#!/usr/bin/env python
"""Per-round floor: a 4000-vertex chain under Bellman-Ford without fusion runs one vertex per
round, so kernel time / rounds is the fixed cost of a round (exploration, not the bench)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

g = gen.chain(4000, np.full(3999, 3, np.uint32))
h = P.SSSP.from_graph(g)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
for pol, par, kw in (("bellman_ford", 0, dict(fuse=False)), ("delta", 1, dict(fuse=False)),
                     ("rho", 1, dict(fuse=False)), ("bellman_ford", 0, dict(snapshot=True))):
    ts = []
    for r in range(5):
        h.run(g.source, pol, par, out=d, **kw)
        ts.append(h.last_stats["kernel_ms"])
    rounds = h.last_stats["rounds"]
    ms = statistics.median(ts)
    _, st, tr, _ = h.run(g.source, pol, par, out=d, trace_cap=8192, **kw)
    ph = {k: float(np.median(tr[k][10:-10])) / 1e3 for k in ("t_theta_ns", "t_extract_ns", "t_relax_ns")}
    print(f"{pol}:{par} {kw}: {ms:.3f} ms, {rounds} rounds, {ms * 1e3 / rounds:.2f} us/round; "
          f"stats-run median phases us {ph}", flush=True)
