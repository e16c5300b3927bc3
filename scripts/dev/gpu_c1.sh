for env in "LINREC_LOCAL=1" "LINREC_LOCAL=0" "LINREC_LOCAL=0 LINREC_NARROW_COLUMNS=1"; do
  echo "== $env"; env $env timeout 300 python scripts/bench_kernel.py --seq-lens 1024,4096 --features 64,256,1024 --out /tmp/x.csv 2>&1 | grep "T="
done
