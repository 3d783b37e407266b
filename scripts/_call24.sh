timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests24.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests24.log
for lib in libsssp.so libsssp_nofuse.so libsssp_f4k.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 3 --configs rmat24,rmat20,grid4096,rgg4m --only rho:262144,rho:131072,bellman_ford:0,delta:8192,rho:4096,rho:16384 --out gpurun_out/sweep_r1t.jsonl --trace gpurun_out/trace_r1t.jsonl > gpurun_out/sweep_r1t_$lib.log 2>&1; echo "== $lib rc=$?"
  grep -E "==|rho|bell|delta|Error" gpurun_out/sweep_r1t_$lib.log
done
