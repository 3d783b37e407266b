set -x
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/gpu_tests6.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gpu_tests6.log
for lib in libsssp.so libsssp_mb1.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 900 python scripts/sweep.py --reps 3 --configs rmat24,grid4096,rgg4m --only rho:262144,rho:4096,bellman_ford:0 --out gpurun_out/sweep_r1e.jsonl --trace gpurun_out/trace_r1e.jsonl > gpurun_out/sweep_r1e_$lib.log 2>&1; echo "sweep $lib rc=$?"
  cat gpurun_out/sweep_r1e_$lib.log
done
CMD="python scripts/run_one.py --config grid1024 --policy rho --param 4096 --reps 2"
timeout 300 $CMD > gpurun_out/run_one.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sssp_round_loop -s 1 -c 1 -o gpurun_out/prof_grid1024 $CMD > gpurun_out/ncu_grid.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_grid.log
