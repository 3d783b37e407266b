#!/usr/bin/env python
"""A/B timing of library variants in one process (exploration, not the bench contract).

  python scripts/ab.py --libs a.so,b.so --config rmat24 --cases rho:262144,delta:131072 --reps 10

Each variant is loaded with its own ctypes handle; runs are interleaved (a, b, a, b, ...)
with an L2 flush before each, so box-to-box and drift effects cancel.  Prints median ms.
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--cases", default="rho:262144")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--kw", default="", help="run options, e.g. fuse_budget=16,small=0")
    a = ap.parse_args()
    import torch
    import gen
    import importlib
    g = gen.make(a.config)
    libs = a.libs.split(",")
    mods = []
    for lib in libs:
        os.environ["SSSP_LIB"] = os.path.join(ROOT, "paper_2105_06145_b200", lib)
        for k in [k for k in sys.modules if k.startswith("paper_2105_06145_b200")]:
            del sys.modules[k]
        mods.append(importlib.import_module("paper_2105_06145_b200"))
    hs = [m.SSSP.from_graph(g) for m in mods]
    d = torch.empty(g.n, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    kw = {k: int(v) for k, v in (x.split("=") for x in a.kw.split(",") if x)}
    for case in a.cases.split(","):
        pol, par = case.split(":")
        par = int(par)
        ts = [[] for _ in libs]
        for h in hs:
            h.run(g.source, pol, par, out=d, **kw)
        for r in range(a.reps):
            for i, h in enumerate(hs):
                flush.zero_()
                h.run(g.source, pol, par, out=d, seed=r, **kw)
                ts[i].append(h.last_stats["kernel_ms"])
        med = [statistics.median(t) for t in ts]
        print(f"{a.config} {pol}:{par} " + "  ".join(f"{l}={m:.3f}ms" for l, m in zip(libs, med))
              + f"  (rel to first: " + " ".join(f"{m / med[0]:.3f}" for m in med) + ")", flush=True)


if __name__ == "__main__":
    main()
