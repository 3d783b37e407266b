timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu_tests29.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests29.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1z.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r1z.log
timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20,grid4096,rgg4m,grid256 --only rho:262144,rho:131072,rho:16384,rho:4096,bellman_ford:0,delta:8192,delta:32768 --out gpurun_out/sweep_r1z.jsonl --trace gpurun_out/trace_r1z.jsonl > gpurun_out/sweep_r1z.log 2>&1; echo "sweep rc=$?"
grep -E "==|rho|bell|delta|Error" gpurun_out/sweep_r1z.log
