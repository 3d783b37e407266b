for lib in libsssp.so libsssp_mb1.so; do
  echo "== $lib"; SSSP_LIB=$PWD/paper_2105_06145_b200/$lib timeout 600 python scripts/round_floor.py 2>&1
done
