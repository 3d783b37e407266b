set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests11.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests11.log
timeout 600 python scripts/round_floor.py 2>&1 | head -3
timeout 900 python scripts/sweep.py --reps 3 --configs rmat24,grid4096,rgg4m,rmat20 --only rho:262144,rho:4096,rho:32768,bellman_ford:0,delta:8192 --out gpurun_out/sweep_r1i.jsonl --trace gpurun_out/trace_r1i.jsonl > gpurun_out/sweep_r1i.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_r1i.log
