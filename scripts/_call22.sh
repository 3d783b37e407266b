for lib in libsssp.so libsssp_k2.so libsssp_k8.so libsssp_l64.so libsssp_l256.so libsssp_e8.so; do
  SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 5 --configs rmat24 --only rho:262144,rho:131072,rho:65536 --out gpurun_out/sweep_r1r.jsonl > gpurun_out/sweep_r1r_$lib.log 2>&1; echo "== $lib rc=$?"
  grep rho gpurun_out/sweep_r1r_$lib.log
done
