#!/usr/bin/env python
"""Small runs of every policy / mode for compute-sanitizer (one tool per call)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402

bad = 0
for name in ("grid64", "rmat12"):
    g = gen.make(name)
    want = oracle.dijkstra(g)
    h = P.SSSP.from_graph(g, validate=True)
    for pol, par in (("rho", 64), ("rho", 1 << 20), ("delta", 3000), ("delta_stepping", 3000), ("bellman_ford", 0),
                     ("dijkstra", 0)):
        for kw in (dict(), dict(snapshot=True), dict(trace_cap=4096, ext_counts=True), dict(nearfar=False),
                   dict(exact=True)):
            r = h.run(g.source, pol, par, **kw)
            d = P.dist_to_u64(r[0] if isinstance(r, tuple) else r)
            if not np.array_equal(d, want):
                bad += 1
                print("MISMATCH", name, pol, par, kw)
    h.close()
import torch  # noqa: E402

keys = torch.tensor([3, 8, 4, 6, 1, 5], dtype=torch.int64, device="cuda")
q = P.LabPQ(keys)
q.update(torch.arange(6))
print("pq", sorted(q.extract(4).tolist()), q.size(), q.select(2, exact=True), q.reduce_min())
print("sanitize_small done, mismatches:", bad)
