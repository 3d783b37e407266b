#!/usr/bin/env python
"""Does a degree-sorted vertex order speed the round loop up?  Builds the rmat24 CSR
relabelled by degree (descending, stable) on the host and times the same policies on the
original and on the relabelled graph (exploration, not the bench)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2105_06145_b200 as P  # noqa: E402


def relabel(g):
    off = g.offsets.astype(np.int64)
    deg = np.diff(off)
    new2old = np.argsort(-deg, kind="stable")
    old2new = np.empty(g.n, np.int64)
    old2new[new2old] = np.arange(g.n)
    ndeg = deg[new2old]
    noff = np.zeros(g.n + 1, np.int64)
    np.cumsum(ndeg, out=noff[1:])
    # gather each new vertex's arc range from the old arrays
    starts = off[new2old]
    rep = np.repeat(starts - noff[:-1], ndeg)
    src_pos = np.arange(g.m, dtype=np.int64) + rep
    nidx = old2new[g.indices[src_pos]].astype(np.int32)
    nw = g.weights[src_pos]
    return gen.Graph(n=g.n, m=g.m, offsets=noff.astype(np.int32), indices=nidx, weights=nw,
                     source=int(old2new[g.source])), old2new


name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
g = gen.make(name)
t0 = time.time()
gr, old2new = relabel(g)
print(f"relabel {time.time() - t0:.1f} s", flush=True)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
hs = {"orig": P.SSSP.from_graph(g), "relabel": P.SSSP.from_graph(gr)}
srcs = {"orig": g.source, "relabel": gr.source}
for pol, par in (("rho", 1 << 18), ("rho", 1 << 21), ("delta", 1 << 17), ("bellman_ford", 0)):
    ts = {k: [] for k in hs}
    for r in range(7):
        for k, h in hs.items():
            flush.zero_()
            h.run(srcs[k], pol, par, out=d, seed=r)
            ts[k].append(h.last_stats["kernel_ms"])
    a, b = statistics.median(ts["orig"]), statistics.median(ts["relabel"])
    print(f"{name} {pol}:{par} orig {a:.3f} ms relabel {b:.3f} ms ({b / a:.3f})", flush=True)
# correctness of the relabelled run
dr = P.dist_to_u64(hs["relabel"].run(gr.source, "rho", 1 << 18, out=d))
do = P.dist_to_u64(hs["orig"].run(g.source, "rho", 1 << 18, out=d))
print("same distances:", bool(np.array_equal(dr[old2new], do)))
