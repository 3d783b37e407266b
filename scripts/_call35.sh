timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests35.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests35.log
for sn in "" "--snapshot"; do
timeout 600 python scripts/sweep.py --reps 5 $sn --configs rmat24,rmat20,grid4096,rgg4m --only rho:262144,rho:131072,rho:16384,bellman_ford:0,delta:32768 --trace gpurun_out/trace_r1eq$sn.jsonl > gpurun_out/sweep_eq$sn.log 2>&1; echo "== $sn"; grep -E "==|rho|bell|delta" gpurun_out/sweep_eq$sn.log
done
