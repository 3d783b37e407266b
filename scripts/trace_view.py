#!/usr/bin/env python
"""Per-round view of sweep.py --trace output: phase times and warp utilisation.

  python scripts/trace_view.py gpurun_out/trace.jsonl [--config rmat24] [--policy rho] [--max 60]
"""
import argparse
import json

NW = 148 * 32  # warps of the default grid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--config", default=None)
    ap.add_argument("--policy", default=None)
    ap.add_argument("--max", type=int, default=60)
    a = ap.parse_args()
    for line in open(a.path):
        d = json.loads(line)
        if a.config and d["config"] != a.config or a.policy and d["policy"] != a.policy:
            continue
        R = d["rounds"]
        n = len(R["qsize"])
        print(f"== {d['config']} {d['policy']} {d['param']} {d.get('tag', '')} rounds={n}")
        tot = {"th": 0.0, "near": 0.0, "A": 0.0, "B": 0.0}
        for i in range(n):
            g = lambda k: R[k][i] if k in R else 0
            th, A, B = g("t_theta_ns") / 1e3, g("t_extract_ns") / 1e3, g("t_relax_ns") / 1e3
            near = g("t_near_ns") / 1e3
            tot["th"] += th; tot["near"] += near; tot["A"] += A; tot["B"] += B
            ua = g("busy_a_ns") / 1e3 / (NW * A) if A else 0
            amax = g("busy_a_max_ns") / 1e3
            if i < a.max:
                print(f"{i:4d} q={g('qsize'):9d} qn={g('qnear'):9d} f={g('fsize'):8d} fu={g('fused'):7d} "
                      f"E={g('edges'):10d} th={th:6.1f} near={near:6.1f} A={A:7.1f} ua={ua:.2f} "
                      f"amax={amax:7.1f} B={B:7.1f} heavy={g('nheavy')}"
                      + (" | per-warp us scan/take/relax/flush/fuse " +
                         " ".join(f"{g(k) / NW / 1.93e3:5.1f}" for k in ("prof_scan", "prof_take", "prof_relax", "prof_flush", "prof_fuse"))
                         + f" fbatches/w {g('prof_fuse_batches') / NW:5.2f} steps/w {g('prof_steps') / NW:5.2f}"
                         + f" us/step {g('prof_step_cyc') / max(1, g('prof_steps')) / 1.93e3:5.2f}"
                         if g("prof_steps") else ""))
        print("totals (us):", {k: round(v, 1) for k, v in tot.items()}, "sum", round(tot["th"] + tot["A"] + tot["B"], 1))


if __name__ == "__main__":
    main()
