for lib in libsssp_a4b1024.so libsssp_a4b1024e2.so libsssp_a2b1024.so libsssp_a2b768m2.so libsssp_a4b512m3.so libsssp_a4b512m2.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20,grid4096 --only rho:262144,bellman_ford:0,rho:16384 --out gpurun_out/sweep_r1x.jsonl > gpurun_out/sweep_r1x_$lib.log 2>&1; echo "== $lib rc=$?"
  grep -E "rho|bell|Error" gpurun_out/sweep_r1x_$lib.log
done
