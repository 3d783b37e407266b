#!/usr/bin/env python
"""Exploration sweep (not the bench contract): time policies/params per config on one GPU.

  python scripts/sweep.py --configs rmat24,grid4096 [--reps 5] [--out gpurun_out/sweep.jsonl]

Per (config, policy, param): median kernel_ms over reps (L2 flushed before each), GTEPS = m/t,
and the stats-run counters -> algorithmic bytes and the HBM roofline fraction.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SWEEPS = {
    "grid256": [("bellman_ford", 0), ("rho", 1 << 10), ("rho", 1 << 12), ("delta", 1 << 13), ("delta", 1 << 15)],
    "rmat20": [("bellman_ford", 0), ("rho", 1 << 13), ("rho", 1 << 15), ("rho", 1 << 17), ("rho", 1 << 19),
               ("rho", 1 << 21), ("delta", 1 << 13), ("delta", 1 << 15), ("delta", 1 << 17)],
    "rgg4m": [("bellman_ford", 0), ("rho", 1 << 11), ("rho", 1 << 12), ("rho", 1 << 14), ("delta", 1 << 8),
              ("delta", 1 << 9), ("delta", 1 << 10)],
    "rmat24": [("bellman_ford", 0), ("rho", 1 << 14), ("rho", 1 << 16), ("rho", 1 << 18), ("rho", 1 << 20),
               ("rho", 1 << 21), ("rho", 1 << 22), ("delta", 1 << 13), ("delta", 1 << 15), ("delta", 1 << 17),
               ("delta", 1 << 19)],
    "grid4096": [("bellman_ford", 0), ("rho", 1 << 12), ("rho", 1 << 13), ("rho", 1 << 15), ("delta", 1 << 13),
                 ("delta", 1 << 14), ("delta", 1 << 15)],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="grid256,rmat20,rgg4m,rmat24,grid4096")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="policy:param,... overrides the built-in sweep")
    ap.add_argument("--snapshot", action="store_true", help="deterministic (snapshot) rounds")
    ap.add_argument("--no-nearfar", action="store_true", help="list all of Q every round (rho)")
    ap.add_argument("--no-fuse", action="store_true", help="no on-the-spot extraction (sparse graphs)")
    ap.add_argument("--fuse-budget", type=int, default=0)
    ap.add_argument("--fuse-depth", type=int, default=0)
    ap.add_argument("--bidir", action="store_true", help="bidirectional relaxation (undirected graphs)")
    ap.add_argument("--trace", default=None, help="append per-round traces of the stats runs here (jsonl)")
    ap.add_argument("--tag", default=os.environ.get("SSSP_LIB", "default"))
    args = ap.parse_args()
    import torch

    import gen
    import paper_2105_06145_b200 as P

    out = open(args.out, "a") if args.out else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name in args.configs.split(","):
        t0 = time.time()
        g = gen.make(name)
        tg = time.time() - t0
        h = P.SSSP.from_graph(g)
        d = torch.empty(g.n, dtype=torch.int64, device="cuda")
        cases = SWEEPS[name]
        if args.only:
            cases = [(c.split(":")[0], int(c.split(":")[1])) for c in args.only.split(",")]
        print(f"== {name}: n={g.n} m={g.m} src={g.source} gen {tg:.1f}s", flush=True)
        for pol, par in cases:
            snap = args.snapshot
            kw = dict(snapshot=snap, nearfar=not args.no_nearfar, max_rounds=200000, fuse=not args.no_fuse,
                      fuse_budget=args.fuse_budget, bidir=args.bidir, fuse_depth=args.fuse_depth)
            for _ in range(2):
                h.run(g.source, pol, par, out=d, **kw)
            ks, rs = [], []
            for r in range(args.reps):
                flush.zero_()
                h.run(g.source, pol, par, out=d, seed=r, **kw)
                ks.append(h.last_stats["kernel_ms"])
                rs.append(h.last_stats["rounds"])
            _, st, tr, _ = h.run(g.source, pol, par, out=d, stats=True, trace_cap=1 << 20 if args.trace else 0, **kw)
            if args.trace and tr is not None:
                with open(args.trace, "a") as f:
                    f.write(json.dumps({"config": name, "policy": pol, "param": par, "tag": args.tag,
                                        "snapshot": snap, "rounds": {k: tr[k].tolist() for k in tr.dtype.names}})
                            + "\n")
            km = statistics.median(ks)
            bt = 8 * st["queue_scanned"] + 8 * st["dense_scanned"] + 8 * st["extracted"] + 16 * st["edges"]
            rec = {"config": name, "policy": pol, "param": par, "tag": args.tag + ("/nonf" if args.no_nearfar else "") + ("/nofuse" if args.no_fuse else "")
                   + (f"/fb{args.fuse_budget}" if args.fuse_budget else "") + (f"/fd{args.fuse_depth}" if args.fuse_depth else "") + ("/bidir" if args.bidir else ""), "snapshot": snap, "kernel_ms": km, "kernel_ms_min": min(ks),
                   "gteps": g.m / km / 1e6, "rounds": statistics.median(rs), "stats_rounds": st["rounds"],
                   "bytes_touched": bt, "touched_gbs": bt / km / 1e6, "frac_6552": bt / km / 1e6 / 6552.6,
                   "edges_per_m": st["edges"] / g.m, "qscan_per_n": st["queue_scanned"] / g.n,
                   "us_per_round": km * 1e3 / max(1, statistics.median(rs)), "grid": st["grid_blocks"],
                   "stats_kernel_ms": st["kernel_ms"]}
            print(f"  {pol:13s} {par:>8d}  {km:9.3f} ms  {rec['gteps']:8.2f} GTEPS  rounds {rec['rounds']:7.0f}  "
                  f"{rec['us_per_round']:7.2f} us/rnd  edges/m {rec['edges_per_m']:6.2f}  "
                  f"touched {rec['touched_gbs']:7.1f} GB/s ({100 * rec['frac_6552']:.1f}%)", flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
                out.flush()
        h.close()
        del g


if __name__ == "__main__":
    main()
