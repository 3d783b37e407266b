timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests23.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests23.log
for lib in libsssp.so libsssp_nol1.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20,grid4096 --only rho:262144,rho:131072,bellman_ford:0,delta:8192,rho:4096 --out gpurun_out/sweep_r1s.jsonl > gpurun_out/sweep_r1s_$lib.log 2>&1; echo "== $lib rc=$?"
  grep -E "==|rho|bell|delta" gpurun_out/sweep_r1s_$lib.log
done
