timeout 600 python scripts/sweep.py --reps 3 --configs rmat24 --only rho:262144 --trace gpurun_out/trace_r1util.jsonl > gpurun_out/sweep_util.log 2>&1; tail -2 gpurun_out/sweep_util.log
