timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests32.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests32.log
for nf in "" "--no-fuse"; do
timeout 600 python scripts/sweep.py --reps 5 $nf --configs rmat24,rmat20,grid4096,rgg4m --only rho:262144,rho:131072,rho:16384,delta:32768,bellman_ford:0 --out gpurun_out/sweep_r1y.jsonl --trace gpurun_out/trace_r1y.jsonl > gpurun_out/sweep_r1y$nf.log 2>&1; echo "== $nf"; grep -E "==|rho|delta|bell|Error" gpurun_out/sweep_r1y$nf.log
done
