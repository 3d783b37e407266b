timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests25.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests25.log
timeout 300 python scripts/sweep.py --reps 3 --configs rmat24 --only rho:262144,bellman_ford:0 > gpurun_out/sweep_r1u_rmat.log 2>&1; grep -E "rho|bell" gpurun_out/sweep_r1u_rmat.log
for fb in 16 64 256; do
  timeout 600 python scripts/sweep.py --reps 3 --fuse-budget $fb --configs grid4096,rgg4m --only rho:4096,rho:16384,rho:65536,delta:8192,delta:32768,bellman_ford:0 --out gpurun_out/sweep_r1u.jsonl > gpurun_out/sweep_r1u_$fb.log 2>&1; echo "== fb $fb rc=$?"
  grep -E "==|rho|bell|delta|Error" gpurun_out/sweep_r1u_$fb.log
done
