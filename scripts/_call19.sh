set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests19.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests19.log
timeout 600 python scripts/sweep.py --reps 3 --configs rmat24,rmat20,grid4096,rgg4m --only rho:65536,rho:131072,rho:262144,rho:524288,rho:1048576,rho:4096,rho:16384 --out gpurun_out/sweep_r1p.jsonl --trace gpurun_out/trace_r1p.jsonl > gpurun_out/sweep_r1p.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_r1p.log
