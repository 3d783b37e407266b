for lib in libsssp.so libsssp_a4b1024.so libsssp_a4b896.so libsssp_a8b640.so libsssp_a4b768.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20 --only rho:262144,bellman_ford:0 --out gpurun_out/sweep_r1w.jsonl > gpurun_out/sweep_r1w_$lib.log 2>&1; echo "== $lib rc=$?"
  grep -E "rho|bell|Error" gpurun_out/sweep_r1w_$lib.log
done
