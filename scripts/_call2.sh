set -x
timeout 1200 python scripts/sweep.py --reps 3 --out gpurun_out/sweep_r1a.jsonl > gpurun_out/sweep_r1a.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/sweep_r1a.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sssp_round_loop -s 3 -c 1 -o gpurun_out/prof_r1a $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
tail -5 gpurun_out/ncu_full.log
