#!/usr/bin/env python
"""Per-round view of runs from seeded random sources (the bench's secondary figure): time,
rounds, arcs scanned / m and the biggest rounds, per source and rho.

  python scripts/multi_source_trace.py --config rmat24 --rhos 262144,2097152 [--sources 10]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat24")
ap.add_argument("--rhos", default="262144,2097152")
ap.add_argument("--sources", type=int, default=10)
a = ap.parse_args()
import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

g = gen.make(a.config)
h = P.SSSP.from_graph(g)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rho in [int(x) for x in a.rhos.split(",")]:
    for v in [g.source] + bench.seeded_sources(g, a.sources):
        h.run(v, "rho", rho, out=d)
        flush.zero_()
        h.run(v, "rho", rho, out=d)
        ms = h.last_stats["kernel_ms"]
        _, st, tr, _ = h.run(v, "rho", rho, out=d, stats=True, trace_cap=4096)
        n = int(st["rounds"])
        big = sorted(((int(tr["edges"][i]), i) for i in range(n)), reverse=True)[:3]
        print(f"{a.config} rho={rho} src={v} deg={int(g.degrees[v])} {ms:.3f} ms rounds={n} "
              f"arcs/m={st['edges'] / g.m:.2f} extracted/n_reached={st['extracted']:.0f} "
              f"biggest rounds (arcs, idx): {big}", flush=True)
