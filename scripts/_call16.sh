set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests16.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests16.log
for lib in libsssp.so libsssp_e4.so libsssp_l32.so libsssp_a4.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 900 python scripts/sweep.py --reps 3 --configs rmat24,rmat20,grid4096,rgg4m --only rho:262144,rho:32768,bellman_ford:0,delta:8192,rho:4096 --out gpurun_out/sweep_r1m.jsonl --trace gpurun_out/trace_r1m.jsonl > gpurun_out/sweep_r1m_$lib.log 2>&1; echo "sweep $lib rc=$?"
  cat gpurun_out/sweep_r1m_$lib.log
done
