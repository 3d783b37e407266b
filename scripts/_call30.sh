set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke30.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke30.log
timeout 900 python bench.py > gpurun_out/bench_default30.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default30.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain30.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/ncu30a.log 2>&1; echo "ncu-launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sssp_round_loop -s 3 -c 1 -o gpurun_out/prof_r1b_rmat24 $CMD > gpurun_out/ncu30b.log 2>&1; echo "ncu-full rc=$?"
