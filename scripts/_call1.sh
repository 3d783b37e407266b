set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config rmat20 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat20.log 2>&1; echo "bench20 rc=$?"
tail -5 gpurun_out/bench_rmat20.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_rmat24.log 2>&1; echo "bench24 rc=$?"
tail -5 gpurun_out/bench_rmat24.log
