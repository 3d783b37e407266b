#!/usr/bin/env python
"""Fill BASELINE.md's results template: 5 configs x {best rho, best Delta*, Bellman-Ford}.

Per (config, policy, param), on one B200:
  GPU   median device time of sssp_run over --reps runs after 3 warm-ups (L2 flushed before each),
        GTEPS = m / t, rounds, B_touched from a stats run (DESIGN.md §5 byte accounting),
        touched GB/s and its fraction of 8 TB/s and of MEASURED_PEAKS.json hbm_gbs,
        distances compared with the oracle's Dijkstra bit for bit;
  CPU   the oracle's binary-heap Dijkstra on 1 host thread (median of 3 on grid256 / rmat20 /
        rgg4m, 1 run on rmat24 / grid4096), MTEPS = m / t.
  ncu   run separately with --ncu-list: one plain launch per case under
        `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,...`;
        --merge-ncu then adds DRAM GB/s, L2 hit % and L2 atomic sectors to the table.

  python scripts/results.py --out gpurun_out/results.jsonl
  ncu --metrics ... --csv --log-file gpurun_out/results_ncu.csv python scripts/results.py --ncu-list
  python scripts/results.py --md profiles/results_r2.md --jsonl gpurun_out/results.jsonl --merge-ncu gpurun_out/results_ncu.csv

(The oracle is called here as the CPU baseline, one of the uses DESIGN.md §3 allows.)
"""
import argparse
import csv
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# best parameters of the parameter study (profiles/param_study_r1.md / param_study_r2.md)
CASES = {
    "grid256": [("rho", 1 << 13), ("delta", 1 << 17), ("bellman_ford", 0)],
    "rmat20": [("rho", 56000), ("rho", 1 << 15), ("delta", 1 << 15), ("bellman_ford", 0)],
    "rgg4m": [("delta", 1 << 12), ("rho", 1 << 14), ("bellman_ford", 0)],
    "rmat24": [("rho", 360000), ("rho", 1 << 18), ("delta", 1 << 17), ("bellman_ford", 0)],
    "grid4096": [("rho", 1 << 14), ("delta", 1 << 17), ("bellman_ford", 0)],
}
LABEL = {"grid256": "C1 grid-256", "rmat20": "C2 R-MAT 20", "rgg4m": "C3 RGG-4M", "rmat24": "C4 R-MAT 24",
         "grid4096": "C5 grid-4096"}
NCU_METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
               "lts__t_sectors_srcunit_tex_op_atom.sum,l1tex__t_sector_hit_rate.pct")


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run_gpu(args):
    import numpy as np
    import torch

    import gen
    import oracle
    import paper_2105_06145_b200 as P

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6552.6))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = open(args.out, "a") if args.out else None
    for name in args.configs.split(","):
        g = gen.make(name)
        h = P.SSSP.from_graph(g)
        d = torch.empty(g.n, dtype=torch.int64, device="cuda")
        # the CPU oracle: ground truth and the 1-thread baseline
        nrep = 3 if name in ("grid256", "rmat20", "rgg4m") else 1
        ts = []
        ref = None
        for _ in range(nrep if not args.ncu_list else 0):
            t0 = time.perf_counter()
            ref = oracle.dijkstra(g)
            ts.append(time.perf_counter() - t0)
        for pol, par in CASES[name]:
            if args.ncu_list:  # one plain launch per case for the ncu metrics pass
                h.run(g.source, pol, par, out=d, max_rounds=300000)
                torch.cuda.synchronize()
                print(json.dumps({"ncu_case": [name, pol, par]}), flush=True)
                continue
            for _ in range(3):
                h.run(g.source, pol, par, out=d, max_rounds=300000)
            ks, rs = [], []
            for r in range(args.reps):
                flush.zero_()
                h.run(g.source, pol, par, out=d, seed=r, max_rounds=300000)
                ks.append(h.last_stats["kernel_ms"])
                rs.append(h.last_stats["rounds"])
            exact = bool(np.array_equal(P.dist_to_u64(d), ref))
            _, st, _, _ = h.run(g.source, pol, par, out=d, stats=True, max_rounds=300000)
            km = statistics.median(ks)
            bt = 8 * st["queue_scanned"] + 8 * st["dense_scanned"] + 8 * st["extracted"] + 16 * st["edges"]
            rec = {"config": name, "n": g.n, "m": g.m, "policy": pol, "param": par, "rounds": statistics.median(rs),
                   "ms": km, "ms_min": min(ks), "reps": args.reps, "gteps": g.m / km / 1e6, "b_touched": bt,
                   "touched_gbs": bt / km / 1e6, "frac_8tb": bt / km / 1e6 / 8000.0, "frac_meas": bt / km / 1e6 / hbm,
                   "hbm_gbs": hbm, "exact": exact, "oracle_s": statistics.median(ts), "oracle_runs": len(ts),
                   "oracle_mteps": g.m / statistics.median(ts) / 1e6, "edges_per_m": st["edges"] / g.m,
                   "cpu": cpu_model(), "host_threads": os.cpu_count()}
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
                out.flush()
        h.close()
        del g


def load_ncu(path):
    """Per case (in launch order) the metrics of its sssp_round_loop launch."""
    rows = {}
    order = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        if "sssp_round_loop" not in row.get("Kernel Name", ""):
            continue
        key = row["ID"]
        if key not in rows:
            rows[key] = {}
            order.append(key)
        v = row["Metric Value"].replace(",", "")
        try:
            rows[key][row["Metric Name"]] = (float(v), row.get("Metric Unit", ""))
        except ValueError:
            pass
    return [rows[k] for k in order]


def to_bytes(val_unit):
    v, u = val_unit
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)


def to_ns(val_unit):
    v, u = val_unit
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)


def write_md(recs, path, ncu=None):
    cases = [(n, p, q) for n in CASES for p, q in CASES[n]]
    if ncu is not None and len(ncu) == len(cases):
        for (n, p, q), m in zip(cases, ncu):
            for r in recs:
                if (r["config"], r["policy"], r["param"]) == (n, p, q):
                    t = to_ns(m["gpu__time_duration.sum"])
                    b = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
                    r["ncu_ms"] = t / 1e6
                    r["ncu_dram_gbs"] = b / t
                    r["ncu_dram_gb"] = b / 1e9
                    r["ncu_l2_hit"] = m["lts__t_sector_hit_rate.pct"][0]
                    r["ncu_l1_hit"] = m.get("l1tex__t_sector_hit_rate.pct", (float("nan"),))[0]
                    r["ncu_atom_sectors"] = m["lts__t_sectors_srcunit_tex_op_atom.sum"][0]
                    r["ncu_atom_per_ns"] = r["ncu_atom_sectors"] / t
    cpu = recs[0]["cpu"] if recs else "?"
    thr = recs[0]["host_threads"] if recs else "?"
    out = ["# Results (BASELINE.md §3 template), B200, one GPU", "",
           f"GPU: median device time of `sssp_run` over {recs[0]['reps'] if recs else '?'} runs after 3 warm-ups, "
           "L2 flushed (256 MiB write) before each; the source is the workload source of each config; "
           "`B_touched` = 8·(ids scanned by Extract + near/far dense-pass reads) + 8·Σ|F_r| + 16·Σ E_r "
           "from a stats run (DESIGN.md §5). "
           f"Fractions against 8 TB/s (north star) and against MEASURED_PEAKS.json `hbm_gbs` "
           f"({recs[0]['hbm_gbs'] if recs else '?'} GB/s, measured copy bandwidth).",
           f"CPU: the oracle's binary-heap Dijkstra (`oracle/`), 1 of {thr} host threads ({cpu}); median of 3 runs "
           "on C1-C3, 1 run on C4/C5; Python `perf_counter` around the call (generation excluded).",
           "ncu: a separate pass, one plain launch per case, `--metrics " + NCU_METRICS + " --clock-control none` "
           "(serialised, cold-cache: its time is not the bench time).", "",
           "| Config | n | m | policy / param | rounds | GPU median ms | GTEPS | B_touched GB | touched GB/s | "
           "% of 8 TB/s | % of meas. | ncu DRAM GB/s | ncu DRAM GB | L2 hit % | L2 atomic sectors/ns | "
           "δ == oracle | oracle s (1 thread) | oracle MTEPS |",
           "|" + "---|" * 18]
    for r in recs:
        par = "-" if r["policy"] == "bellman_ford" else (
            f"2^{r['param'].bit_length() - 1}" if r["param"] & (r["param"] - 1) == 0 else f"{r['param']:,}")
        nc = lambda k, f: (f.format(r[k]) if k in r else "-")  # noqa: E731
        out.append(f"| {LABEL[r['config']]} | {r['n']:,} | {r['m']:,} | {r['policy']} {par} | {r['rounds']:.0f} | "
                   f"{r['ms']:.3f} | {r['gteps']:.2f} | {r['b_touched'] / 1e9:.3f} | {r['touched_gbs']:.0f} | "
                   f"{100 * r['frac_8tb']:.1f} | {100 * r['frac_meas']:.1f} | {nc('ncu_dram_gbs', '{:.0f}')} | "
                   f"{nc('ncu_dram_gb', '{:.3f}')} | {nc('ncu_l2_hit', '{:.1f}')} | {nc('ncu_atom_per_ns', '{:.2f}')} | "
                   f"{'yes' if r['exact'] else 'NO'} | {r['oracle_s']:.3f} | {r['oracle_mteps']:.1f} |")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(CASES))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--ncu-list", action="store_true", help="one plain launch per case (run under ncu)")
    ap.add_argument("--md", default=None)
    ap.add_argument("--jsonl", default=None)
    ap.add_argument("--merge-ncu", default=None)
    args = ap.parse_args()
    if args.md:
        recs = [json.loads(ln) for ln in open(args.jsonl)]
        write_md(recs, args.md, load_ncu(args.merge_ncu) if args.merge_ncu else None)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
