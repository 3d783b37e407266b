timeout 1800 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu_tests40.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests40.log
timeout 300 python scripts/sweep.py --reps 5 --configs rmat24 --only rho:262144 > gpurun_out/sweep40.log 2>&1; grep rho gpurun_out/sweep40.log
