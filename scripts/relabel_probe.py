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


def relabel(g, hot=None):
    off = g.offsets.astype(np.int64)
    deg = np.diff(off)
    order = np.argsort(-deg, kind="stable")
    if hot is None:  # full degree order
        new2old = order
    elif hot == 0:  # isolated vertices last, everything else in its original order
        new2old = np.concatenate([np.flatnonzero(deg > 0), np.flatnonzero(deg == 0)])
    else:  # the library's scheme: top `hot` to 0.., displaced low ids to the freed ids
        new2old = np.arange(g.n)
        top = order[:hot]
        is_hot = np.zeros(g.n, bool)
        is_hot[top] = True
        freed = np.sort(top[top >= hot])
        displaced = np.flatnonzero(~is_hot[:hot])
        new2old[:hot] = top
        new2old[freed] = displaced
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
gp, _ = relabel(g, hot=g.n // 16)
gc, _ = relabel(g, hot=0)
print(f"relabel {time.time() - t0:.1f} s", flush=True)
d = torch.empty(g.n, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
hs = {"orig": P.SSSP.from_graph(g, relabel=False), "relabel": P.SSSP.from_graph(gr, relabel=False),
      "partial": P.SSSP.from_graph(gp, relabel=False), "compact": P.SSSP.from_graph(gc, relabel=False)}
srcs = {"orig": g.source, "relabel": gr.source, "partial": gp.source, "compact": gc.source}
for pol, par in (("rho", 1 << 18), ("rho", 1 << 21), ("delta", 1 << 17), ("bellman_ford", 0)):
    ts = {k: [] for k in hs}
    for r in range(7):
        for k, h in hs.items():
            flush.zero_()
            h.run(srcs[k], pol, par, out=d, seed=r)
            ts[k].append(h.last_stats["kernel_ms"])
    med = {k: statistics.median(v) for k, v in ts.items()}
    print(f"{name} {pol}:{par} " + " ".join(f"{k} {v:.3f} ms ({v / med['orig']:.3f})" for k, v in med.items()), flush=True)
# correctness of the relabelled run
dr = P.dist_to_u64(hs["relabel"].run(gr.source, "rho", 1 << 18, out=d))
do = P.dist_to_u64(hs["orig"].run(g.source, "rho", 1 << 18, out=d))
print("same distances:", bool(np.array_equal(dr[old2new], do)))
