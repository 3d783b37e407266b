set -x
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain21.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu21a.log 2>&1; echo "ncu-launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sssp_round_loop -s 3 -c 1 -o gpurun_out/prof_r1_rmat24 $CMD > gpurun_out/ncu21b.log 2>&1; echo "ncu-full rc=$?"
tail -3 gpurun_out/ncu21b.log
