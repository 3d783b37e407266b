timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu_tests26.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests26.log
timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20,grid4096,rgg4m,grid256 --only rho:262144,rho:16384,rho:4096,bellman_ford:0,delta:8192,delta:32768 --out gpurun_out/sweep_r1v.jsonl --trace gpurun_out/trace_r1v.jsonl > gpurun_out/sweep_r1v.log 2>&1; echo "sweep rc=$?"
grep -E "==|rho|bell|delta|Error" gpurun_out/sweep_r1v.log
