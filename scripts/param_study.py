#!/usr/bin/env python
"""SURVEY f-3: rho / Delta sweeps on the five configs (paper Fig. rho-time, Fig.
intro:delta P:493-512).  Runs scripts/sweep.py-style timing and writes a markdown table.

  python scripts/param_study.py --out gpurun_out/param_study.jsonl --md gpurun_out/param_study.md
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RHOS = [1 << k for k in range(10, 24, 1)]
DELTAS = {"grid256": [1 << k for k in range(11, 20)], "grid4096": [1 << k for k in range(11, 20)],
          "rgg4m": [1 << k for k in range(6, 15)], "rmat20": [1 << k for k in range(10, 20)],
          "rmat24": [1 << k for k in range(8, 21)]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="grid256,rmat20,rgg4m,rmat24,grid4096")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/param_study.jsonl")
    ap.add_argument("--md", default="gpurun_out/param_study.md")
    args = ap.parse_args()
    import torch

    import gen
    import paper_2105_06145_b200 as P

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    recs = []
    for name in args.configs.split(","):
        g = gen.make(name)
        h = P.SSSP.from_graph(g)
        d = torch.empty(g.n, dtype=torch.int64, device="cuda")
        cases = [("bellman_ford", 0)] + [("rho", r) for r in RHOS] + [("delta", x) for x in DELTAS[name]] + \
                [("delta_stepping", x) for x in DELTAS[name][::2]]
        for pol, par in cases:
            h.run(g.source, pol, par, out=d, max_rounds=300000)
            ks, rs = [], []
            for r in range(args.reps):
                flush.zero_()
                h.run(g.source, pol, par, out=d, seed=r, max_rounds=300000)
                ks.append(h.last_stats["kernel_ms"])
                rs.append(h.last_stats["rounds"])
            _, st, _, _ = h.run(g.source, pol, par, out=d, stats=True, max_rounds=300000)
            km = statistics.median(ks)
            rec = {"config": name, "policy": pol, "param": par, "ms": km, "gteps": g.m / km / 1e6,
                   "rounds": statistics.median(rs), "edges_per_m": st["edges"] / g.m}
            recs.append(rec)
            print(json.dumps(rec), flush=True)
        h.close()
    with open(args.out, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    write_md(recs, args.md)


def write_md(recs, path):
    out = ["# Parameter study (SURVEY f-3), B200, one source per config (the workload source)", "",
           "Median device time of `sssp_run` over 3 runs (L2 flushed before each), default live rounds.", ""]
    for name in dict.fromkeys(r["config"] for r in recs):
        rs = [r for r in recs if r["config"] == name]
        out += [f"## {name}", "", "| policy | param | ms | GTEPS | rounds | arcs scanned / m |", "|---|---|---|---|---|---|"]
        best = {}
        for r in rs:
            b = best.get(r["policy"])
            if b is None or r["ms"] < b["ms"]:
                best[r["policy"]] = r
        for r in rs:
            mark = " **best**" if best[r["policy"]] is r else ""
            par = "-" if r["policy"] == "bellman_ford" else (f"2^{r['param'].bit_length() - 1}")
            out.append(f"| {r['policy']}{mark} | {par} | {r['ms']:.3f} | {r['gteps']:.2f} | {r['rounds']:.0f} | "
                       f"{r['edges_per_m']:.2f} |")
        out.append("")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
