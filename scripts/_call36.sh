for lib in libsssp.so libsssp_c16.so libsssp_c1.so libsssp_c64.so; do
SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/sweep.py --reps 5 --configs rmat24,rmat20,grid4096,rgg4m --only rho:262144,rho:16384,bellman_ford:0,delta:32768 > gpurun_out/sweep_c_$lib.log 2>&1; echo "== $lib"; grep -E "rho|bell|delta" gpurun_out/sweep_c_$lib.log
done
