timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests37.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests37.log
for fb in 64 1024 4096; do
timeout 600 python scripts/sweep.py --reps 3 --fuse-budget $fb --configs grid4096,rgg4m,grid256 --only rho:4096,rho:16384,rho:65536,delta:32768,delta:131072,bellman_ford:0 > gpurun_out/sweep_fb$fb.log 2>&1; echo "== fb $fb"; grep -E "==|rho|bell|delta" gpurun_out/sweep_fb$fb.log
done
