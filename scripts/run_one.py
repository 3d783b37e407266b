#!/usr/bin/env python
"""One config/policy/param: a few sssp_run launches (for ncu / sanitizer captures). Not the bench contract."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="grid1024")
ap.add_argument("--policy", default="rho")
ap.add_argument("--param", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--snapshot", action="store_true")
a = ap.parse_args()
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

g = gen.make(a.config)
h = P.SSSP.from_graph(g)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
for r in range(a.reps):
    h.run(g.source, a.policy, a.param, out=d, snapshot=a.snapshot)
    print(a.config, a.policy, a.param, h.last_stats["kernel_ms"], "ms", h.last_stats["rounds"], "rounds", flush=True)
