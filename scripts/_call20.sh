set -x
timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu_tests20.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests20.log
timeout 600 python scripts/sweep.py --reps 3 --configs rmat24,grid4096 --only rho:262144,rho:131072,rho:4096 --out gpurun_out/sweep_r1q.jsonl --trace gpurun_out/trace_r1q.jsonl > gpurun_out/sweep_r1q.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_r1q.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1q.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench_r1q.log
