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
    ap.add_argument("--traces", default=None, help="also record per-step traces of rho / Delta* / BF (jsonl)")
    ap.add_argument("--trace-configs", default="rmat24,rgg4m,grid4096")
    ap.add_argument("--from-jsonl", action="store_true", help="only rewrite --md from --out (and --traces)")
    args = ap.parse_args()
    if args.from_jsonl:
        write_md([json.loads(ln) for ln in open(args.out)], args.md, args.traces)
        return
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
        if args.traces and name in args.trace_configs.split(","):
            # visited vertices per step (paper Fig. visted-per-step) at the best rho / Delta*
            mine = [r for r in recs if r["config"] == name]
            for pol in ("rho", "delta", "bellman_ford"):
                b = min((r for r in mine if r["policy"] == pol), key=lambda r: r["ms"])
                _, st, tr, _ = h.run(g.source, pol, b["param"], out=d, stats=True, trace_cap=1 << 20,
                                     max_rounds=300000)
                with open(args.traces, "a") as f:
                    f.write(json.dumps({"config": name, "n": g.n, "m": g.m, "policy": pol, "param": b["param"],
                                        "ms": b["ms"], "fsize": tr["fsize"].tolist(), "edges": tr["edges"].tolist(),
                                        "qsize": tr["qsize"].tolist(), "fused": tr["fused"].tolist()}) + "\n")
        h.close()
    with open(args.out, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    write_md(recs, args.md, args.traces)


def fixed_rho(recs):
    """One rho for every config (the paper's PQ-rho-fix): the rho of the sweep
    with the smallest geometric-mean slowdown against each config's best rho."""
    import math

    rho = [r for r in recs if r["policy"] == "rho"]
    cfgs = list(dict.fromkeys(r["config"] for r in rho))
    best = {c: min((r for r in rho if r["config"] == c), key=lambda r: r["ms"]) for c in cfgs}
    rows = []
    for p in sorted(set(r["param"] for r in rho)):
        at = {c: next((r for r in rho if r["config"] == c and r["param"] == p), None) for c in cfgs}
        if any(v is None for v in at.values()):
            continue
        loss = {c: at[c]["ms"] / best[c]["ms"] for c in cfgs}
        geo = math.exp(sum(math.log(x) for x in loss.values()) / len(loss))
        rows.append((geo, max(loss.values()), p, loss))
    rows.sort(key=lambda t: t[0])
    return cfgs, best, rows


def step_table(t, bins=20):
    """Visited vertices (|F_r|, fusion included) and arcs per step; long runs grouped into bins."""
    f, e, q = t["fsize"], t["edges"], t["qsize"]
    R = len(f)
    out = [f"### {t['config']} {t['policy']}" + ("" if t["policy"] == "bellman_ford" else
                                                 f" 2^{t['param'].bit_length() - 1}") +
           f" ({R} steps, {t['ms']:.3f} ms; visited / n = {sum(f) / t['n']:.2f}, arcs / m = {sum(e) / t['m']:.2f})", ""]
    if R <= 40:
        out += ["| step | \\|Q\\| | visited \\|F\\| | arcs |", "|---|---|---|---|"]
        out += [f"| {i + 1} | {q[i]:,} | {f[i]:,} | {e[i]:,} |" for i in range(R)]
    else:
        k = (R + bins - 1) // bins
        out += ["| steps | mean \\|Q\\| | visited (sum) | visited (max step) | arcs (sum) |", "|---|---|---|---|---|"]
        for s in range(0, R, k):
            sl = slice(s, min(R, s + k))
            out.append(f"| {s + 1}-{min(R, s + k)} | {sum(q[sl]) / len(q[sl]):,.0f} | {sum(f[sl]):,} | "
                       f"{max(f[sl]):,} | {sum(e[sl]):,} |")
    return out + [""]


def write_md(recs, path, traces=None):
    out = ["# Parameter study (SURVEY f-3), B200, one source per config (the workload source)", "",
           "Median device time of `sssp_run` over 3 runs (L2 flushed before each), default live rounds.", ""]
    cfgs, best, rows = fixed_rho(recs)
    out += ["## Summary: best parameter per policy (ms, lower is better)", "",
            "| config | BF | rho best (rho) | rho fixed" + (f" (2^{rows[0][2].bit_length() - 1})" if rows else "") +
            " | Delta* best (Delta) | Delta-stepping best (Delta) |", "|---|---|---|---|---|---|"]
    for c in dict.fromkeys(r["config"] for r in recs):
        def bestof(pol):
            rs = [r for r in recs if r["config"] == c and r["policy"] == pol]
            return min(rs, key=lambda r: r["ms"]) if rs else None
        cell = lambda r: "-" if r is None else (f"{r['ms']:.2f}" if r["policy"] == "bellman_ford" else  # noqa: E731
                                                f"{r['ms']:.2f} (2^{r['param'].bit_length() - 1})")
        fx = next((r for r in recs if rows and r["config"] == c and r["policy"] == "rho" and r["param"] == rows[0][2]), None)
        out.append(f"| {c} | {cell(bestof('bellman_ford'))} | {cell(bestof('rho'))} | "
                   f"{'-' if fx is None else format(fx['ms'], '.2f')} | {cell(bestof('delta'))} | "
                   f"{cell(bestof('delta_stepping'))} |")
    out.append("")
    if rows:
        geo, mx, p, loss = rows[0]
        out += [f"## One fixed GPU rho for all configs (PQ-rho-fix analogue, P:1575, P:1601)", "",
                f"rho = 2^{p.bit_length() - 1} has the smallest geometric-mean slowdown against each config's best "
                f"rho ({geo:.3f}x; worst {mx:.2f}x). Candidates ranked:", "",
                "| rho | geo-mean loss | worst | " + " | ".join(cfgs) + " |", "|---|---|---|" + "---|" * len(cfgs)]
        for geo_, mx_, p_, loss_ in rows[:6]:
            out.append(f"| 2^{p_.bit_length() - 1} | {geo_:.3f} | {mx_:.2f} | " +
                       " | ".join(f"{loss_[c]:.2f}" for c in cfgs) + " |")
        out += ["", "Best rho per config: " + ", ".join(f"{c} 2^{best[c]['param'].bit_length() - 1} "
                                                        f"({best[c]['ms']:.3f} ms)" for c in cfgs) + ".", ""]
    if traces and os.path.exists(traces):
        out += ["## Visited vertices per step (paper Fig. visted-per-step, P:1653-1678)", "",
                "From the trace rows of a stats run at each policy's best parameter. Visited = |F_r|, the vertices "
                "extracted in step r (vertices relaxed on the spot by fusion included).", ""]
        for ln in open(traces):
            out += step_table(json.loads(ln))
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
