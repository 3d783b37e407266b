set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests10.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests10.log
for lib in libsssp.so libsssp_b768.so libsssp_b1024.so; do
  echo "== $lib"; SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/round_floor.py 2>&1 | head -3
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 900 python scripts/sweep.py --reps 3 --configs rmat24,grid4096,rgg4m,rmat20 --only rho:262144,rho:4096,rho:32768,bellman_ford:0,delta:8192 --out gpurun_out/sweep_r1h.jsonl --trace gpurun_out/trace_r1h.jsonl > gpurun_out/sweep_r1h_$lib.log 2>&1; echo "sweep $lib rc=$?"
  cat gpurun_out/sweep_r1h_$lib.log
done
