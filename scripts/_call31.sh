timeout 1800 python -m pytest tests -m "gpu" -x -q > gpurun_out/gpu_tests31.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/gpu_tests31.log
timeout 600 python scripts/sweep.py --reps 3 --configs rmat24,rmat20,grid4096,rgg4m --only delta_stepping:8192,delta_stepping:32768,delta:32768 > gpurun_out/sweep_r1ds.log 2>&1; grep -E "==|delta" gpurun_out/sweep_r1ds.log
