set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests8.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests8.log
for lib in libsssp.so libsssp_mb1.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 900 python scripts/sweep.py --reps 3 --configs rmat24,grid4096,rgg4m,rmat20 --only rho:262144,rho:4096,rho:32768,bellman_ford:0,delta:8192 --out gpurun_out/sweep_r1g.jsonl --trace gpurun_out/trace_r1g.jsonl > gpurun_out/sweep_r1g_$lib.log 2>&1; echo "sweep $lib rc=$?"
  cat gpurun_out/sweep_r1g_$lib.log
done
