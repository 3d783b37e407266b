#!/usr/bin/env python
"""Benchmark: SSSP GTEPS of the stepping-algorithm hot path on B200 (BASELINE.json metric).

A step = one sssp_run (Alg. 1, all rounds) from the workload's source on a resident
graph; GTEPS = m / device time per source.  Default workload (N=1): R-MAT scale 24
(BASELINE.json configs[3], the config the north-star target is quoted on), rho-stepping.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat24] [--policy rho] [--param P]
  python bench.py --impl reference ...   # the CPU oracle arm (bounded Dijkstra samples, rank 0 only)

Multi-GPU (torchrun): the path has no exchange step; every rank runs an independent
replica (its own source on a full copy of the graph) -> "scaling": "weak", no collective
in the timed region other than the barriers and the max-over-ranks reduction.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# rho = 360,000: the tuned rho of rmat24 (PQ-rho-best).  The power-of-two study puts the best rho at
# 2^18; a finer sweep between 2^18 and the cliff keeps gaining (profiles/param_study_r2_fine.md:
# 2^18 3.75 ms, 360,000 3.63 ms, 400,000 3.60 ms over 20 sampling seeds each).  The cliff is the
# source's degree, 406,678 = |Q_2|: from there on |Q_2| <= rho makes theta_2 = +inf, the whole
# first frontier is extracted with tentative keys and every arc is relaxed 1.56 times (4.77 ms at
# 450,000, as at 2^19).  360,000 leaves an 11 % margin below it.
DEFAULT_PARAM = {"rho": 360000, "delta": 1 << 15, "bellman_ford": 0, "dijkstra": 0}
PAPER_RHO_FIX = 1 << 21  # PQ-rho-fix on scale-free graphs
CONFIG_DESC = {
    "grid256": "2D 4-neighbour grid 256x256, weights U[1,65535], source 0",
    "rmat20": "R-MAT scale 20, ef 16 (.57,.19,.19,.05), symmetrised+dedup, weights U[1,2^18), source = max degree",
    "rgg4m": "random geometric 4-NN graph, 2^22 points, weight round(len*1e6)+1, source nearest (0.5,0.5)",
    "rmat24": "R-MAT scale 24, ef 16 (.57,.19,.19,.05), symmetrised+dedup, weights log-uniform [1,2^20), "
              "source = max degree",
    "grid4096": "2D 4-neighbour grid 4096x4096, weights U[1,65535], source 0 (corner)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--policy", default="rho", choices=["rho", "delta", "bellman_ford", "dijkstra"])
    ap.add_argument("--param", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-arc-budget", type=int, default=-1,
                    help="cpu_baseline: stop the oracle after this many arc scans (-1: full run)")
    ap.add_argument("--sources", type=int, default=10, help="secondary figure: seeded non-isolated sources")
    ap.add_argument("--rho-fix-steps", type=int, default=5,
                    help="secondary figure: timed runs at the paper's fixed rho = 2^21 (0 = skip)")
    ap.add_argument("--no-flush", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_traffic(config, policy):
    """dram bytes per launch of the round-loop kernel from a committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(f"{config}/{policy}")
        return (int(e["dram_bytes_per_launch"]), e.get("source")) if e else (None, None)
    except Exception:
        return None, None


def make_graph(name):
    import gen

    if name not in gen.CONFIGS:
        raise SystemExit(f"unknown config {name}; choose from {sorted(gen.CONFIGS)}")
    return gen.make(name)


def replica_source(g, rank):
    """Source of a replica: rank 0 runs the workload's source, rank r > 0 a seeded random
    non-isolated vertex (independent single-source problems: no data-path collective)."""
    import numpy as np

    if rank == 0:
        return int(g.source)
    rs = np.random.default_rng(1000 + rank)
    deg = g.degrees
    while True:
        v = int(rs.integers(0, g.n))
        if deg[v] > 0:
            return v


def max_over_ranks(x, ws, dist=None, device=None):
    """Max of a per-rank float over the job (the timing rule: the slowest rank decides)."""
    if ws <= 1:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload_config(args, g, source, param, ws):
    """The `config` object, identical in both arms (ours and --impl reference)."""
    return {"workload": f"{args.config}: {CONFIG_DESC.get(args.config, args.config)}",
            "n": g.n, "m": g.m, "source": source, "policy": args.policy, "param": param,
            "parallelism": f"replicas x{ws} (independent sources, no collective)",
            "l2": "GPU arm: L2 flushed between timed steps (256 MiB write); reference arm: host CPU"}


def emit(obj):
    print(json.dumps(obj), flush=True)


# ----------------------------------------------------------------------------- CPU oracle arms
def cpu_oracle_sample(g, source, arc_budget):
    """The oracle (plain binary-heap Dijkstra, 1 thread) on the same graph, stopped after
    `arc_budget` arc scans (arc_budget >= m: the full run)."""
    import oracle

    t0 = time.perf_counter()
    scanned, settled = oracle.dijkstra_budget(g, source, arc_budget)
    dt = time.perf_counter() - t0
    return scanned, settled, dt


def seeded_sources(g, k, seed=2105):
    """k seeded random non-isolated sources (the paper averages 10 sources)."""
    import numpy as np

    nz = np.flatnonzero(g.degrees > 0)
    rs = np.random.default_rng(seed)
    return [int(v) for v in rs.choice(nz, size=min(k, len(nz)), replace=False)]


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle arm
    g = make_graph(args.config)
    param = DEFAULT_PARAM[args.policy] if args.param is None else args.param
    # each timed step a bounded sample sized so that K steps scan ~10 m arcs in total (a full
    # run per step for K <= 10; ~20 s per full run on rmat24): the whole arm ends in a few
    # minutes.  Warm-up steps (untimed) are 1 % samples: they only warm the host caches.
    budget = g.m if args.steps <= 10 else g.m * 10 // args.steps
    for _ in range(args.warmup):
        cpu_oracle_sample(g, g.source, max(1, g.m // 100))
    tot_arcs, tot_t, settled = 0, 0.0, 0
    for _ in range(args.steps):
        a, s, dt = cpu_oracle_sample(g, g.source, budget)
        tot_arcs += a
        tot_t += dt
        settled = s
    gteps = tot_arcs / tot_t / 1e9
    sample = (f"binary-heap Dijkstra (oracle/, 1 host thread of {os.cpu_count()}) from the workload source, "
              + ("full run per step" if budget >= g.m else f"stopped after {budget} arc scans per step")
              + f" ({settled} vertices settled); GTEPS = arcs scanned / time")
    emit({"impl": "reference", "metric": "SSSP GTEPS (m / device time per source)", "value": gteps,
          "unit": "GTEPS", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
          "vs_baseline": None, "dtype": "u64", "data": "synthetic",
          "config": workload_config(args, g, g.source, param, ws),
          "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": 1, "kind": "oracle", "sample": sample,
                           "host_threads": os.cpu_count()},
          "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2105_06145_b200 as P

    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    param = DEFAULT_PARAM[args.policy] if args.param is None else args.param

    t_gen = time.perf_counter()
    g = make_graph(args.config)
    t_gen = time.perf_counter() - t_gen
    source = replica_source(g, rank)
    h = P.SSSP.from_graph(g, device=dev)
    stream = h.stream
    out = torch.empty(g.n, dtype=torch.int64, device=dev)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        h.run(source, args.policy, param, out=out, seed=args.seed)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    barrier()
    step_ms, kern_ms, rounds = [], [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()  # evict L2 (126 MB) between timed steps; not inside the events
        ev0.record(stream)
        h.run(source, args.policy, param, out=out, seed=args.seed + k)
        ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        kern_ms.append(h.last_stats["kernel_ms"])
        rounds.append(h.last_stats["rounds"])
    barrier()
    total_ms = max_over_ranks(sum(step_ms), ws, dist, dev)
    clocks = sampler.stop()
    ms_per_step = total_ms / args.steps
    value = ws * g.m / (ms_per_step * 1e-3) / 1e9

    # end-to-end: the public host-buffer call for many sources, sssp_run_batch_host: every
    # step's n distances are copied to pinned host memory (the read-back of step i overlaps
    # the run of step i+1 on a second stream); the graph is resident and the source is
    # passed by value (4 bytes)
    host = torch.empty((args.steps, g.n), dtype=torch.int64, pin_memory=True)
    h.run_batch_host([source] * min(2, args.steps), args.policy, param, host[:min(2, args.steps)])
    barrier()
    t0 = time.perf_counter()
    h.run_batch_host([source] * args.steps, args.policy, param, host)
    e2e_s = max_over_ranks(time.perf_counter() - t0, ws, dist, dev)
    e2e = ws * g.m * args.steps / e2e_s / 1e9

    # algorithmic bytes: counters runs (the STATS variant
    # of the kernel) with the SAME seeds as the timed steps, averaged, so that bytes and time
    # describe the same rounds (sampled theta depends on the seed)
    bts, sts = [], []
    for k in range(args.steps):
        _, st, _, _ = h.run(source, args.policy, param, out=out, stats=True, seed=args.seed + k)
        bts.append(8 * st["queue_scanned"] + 8 * st["dense_scanned"] + 8 * st["extracted"] + 16 * st["edges"])
        sts.append(st)
    b_touched = statistics.mean(bts)
    kern_avg = statistics.mean(kern_ms)

    # secondary figure: seeded non-isolated sources (the paper averages 10 sources)
    multi = None
    if args.sources > 0:
        ms_src = []
        for v in seeded_sources(g, args.sources):
            h.run(v, args.policy, param, out=out, seed=args.seed)
            if flush is not None:
                flush.zero_()
            h.run(v, args.policy, param, out=out, seed=args.seed)
            ms_src.append(h.last_stats["kernel_ms"])
        multi = {"sources": len(ms_src), "kernel_ms_mean": statistics.mean(ms_src),
                 "kernel_ms_min": min(ms_src), "kernel_ms_max": max(ms_src),
                 "gteps_mean": statistics.mean(g.m / t / 1e6 for t in ms_src),
                 "note": "seeded random non-isolated sources (numpy default_rng(2105)), one warm run then one "
                         "timed run each after an L2 flush; GTEPS = m / time"}
    peak, peak_src = load_peaks()
    achieved = b_touched / (kern_avg * 1e-3) / 1e9
    # distance bytes of S0 (init) and S6 (output), which are inside the timed launch but not in
    # SURVEY 8(d)'s B_touched: reported separately, never folded into `frac`
    nz = int((g.degrees > 0).sum())
    compacted = g.m >= 20 * g.n and g.n >= 64 and g.n - nz >= g.n // 16  # run.cu may_compact / build_compaction
    n_run = nz if compacted else g.n
    io_bytes = 8 * n_run + 8 * n_run + (8 * g.n if compacted else 0)

    # secondary figure: the paper's fixed parameter, PQ-rho-fix = 2^21 on scale-free graphs
    # (P:1575), next to the tuned rho of the headline (PQ-rho-best): same timing and
    # byte accounting, fewer steps
    rho_fix = None
    if args.policy == "rho" and param != PAPER_RHO_FIX and args.rho_fix_steps > 0:
        for _ in range(3):
            h.run(source, "rho", PAPER_RHO_FIX, out=out, seed=args.seed)
        ms_fix, b_fix, r_fix = [], [], []
        for k in range(args.rho_fix_steps):
            if flush is not None:
                flush.zero_()
            h.run(source, "rho", PAPER_RHO_FIX, out=out, seed=args.seed + k)
            ms_fix.append(h.last_stats["kernel_ms"])
            r_fix.append(h.last_stats["rounds"])
        for k in range(args.rho_fix_steps):
            _, st, _, _ = h.run(source, "rho", PAPER_RHO_FIX, out=out, stats=True, seed=args.seed + k)
            b_fix.append(8 * st["queue_scanned"] + 8 * st["dense_scanned"] + 8 * st["extracted"] + 16 * st["edges"])
        t_fix, bt_fix = statistics.mean(ms_fix), statistics.mean(b_fix)
        a_fix = bt_fix / (t_fix * 1e-3) / 1e9
        rho_fix = {"rho": PAPER_RHO_FIX, "steps": args.rho_fix_steps, "kernel_ms_mean": t_fix,
                   "gteps": g.m / t_fix / 1e6, "rounds_median": statistics.median(r_fix),
                   "algorithmic_bytes_per_launch": bt_fix, "achieved_gbs": a_fix, "frac": a_fix / peak,
                   "frac_of_8TBps": a_fix / 8000.0,
                   "note": "the paper's fixed rho = 2^21 (PQ-rho-fix, P:1575, P:1601) on the same workload and "
                           "source: more arcs re-relaxed per run (bytes up), fewer rounds; the headline uses the "
                           "tuned rho (PQ-rho-best)"}
    traffic, traffic_src = load_traffic(args.config, args.policy)

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        budget = g.m if args.cpu_arc_budget < 0 else min(g.m, args.cpu_arc_budget)
        scanned, settled, dt = cpu_oracle_sample(g, source, budget)
        full = budget >= g.m
        cpu = {"value": (g.m if full else scanned) / dt / 1e9, "unit": "GTEPS", "cores": 1, "kind": "oracle",
               "host_threads": os.cpu_count(), "seconds": dt,
               "sample": (f"full binary-heap Dijkstra (oracle/, 1 host thread of {os.cpu_count()}) from the same "
                          f"source: {settled} vertices settled, {scanned} arcs scanned, {dt:.1f} s; GTEPS = m / time"
                          if full else
                          f"binary-heap Dijkstra (oracle/, 1 host thread of {os.cpu_count()}) from the same source, "
                          f"stopped after {scanned} arc scans ({settled} vertices settled), {dt:.1f} s")}
    emit({"metric": "SSSP GTEPS (m / device time per source)", "value": value, "unit": "GTEPS", "n_gpus": ws,
          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
          "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
          "config": workload_config(args, g, g.source, param, ws),
          "multi_source": multi,
          "rho_fix": rho_fix,
          "run": {"source_this_rank": source, "l2_flushed": flush is not None,
                  "rounds_median": statistics.median(rounds), "kernel_ms_mean": kern_avg,
                  "grid": [st["grid_blocks"], st["block_threads"]], "gen_s": round(t_gen, 1)},
          "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                       "traffic": traffic, "peak_source": peak_src,
                       "frac_of_8TBps": achieved / 8000.0,
                       "init_output_distance_bytes": io_bytes,
                       "frac_of_8TBps_incl_init_output": (b_touched + io_bytes) / (kern_avg * 1e-3) / 1e9 / 8000.0,
                       "init_output_note": "secondary: B_touched plus the distance bytes of S0 / S6 inside the same launch "
                                           "(init writes 8*n_run, the output pass reads 8*n_run and writes 8*n); SURVEY "
                                           "8(d)'s formula, which `achieved` and `frac` follow, leaves them out",
                       "algorithmic_bytes_per_launch": b_touched,
                       "bytes_formula": "8*(ids scanned by Extract + vertices read by near/far dense passes) + 8*sum|F_r| "
                                           "+ 16*sum E_r (SURVEY 8(d) B_touched; DESIGN.md §5), mean over counters "
                                           "runs with the timed steps' seeds",
                       "traffic_source": traffic_src},
          "cpu_baseline": cpu,
          "e2e": {"value": e2e, "unit": "GTEPS", "h2d_bytes_per_step": 4, "d2h_bytes_per_step": 8 * g.n,
                  "note": "sssp_run_batch_host over the timed steps: graph resident (created once), source "
                          "passed by value, n uint64 distances copied to pinned host memory per step, the copy "
                          "of step i overlapping the run of step i+1; host wall clock"},
          "gpu_launches": args.steps,
          "clocks": clocks,
          "counters": {k: statistics.mean(x[k] for x in sts) for k in
                       ("rounds", "extracted", "edges", "succ", "inserts", "queue_scanned", "dense_scanned",
                        "max_queue", "max_frontier")}})
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
