mkdir -p gpurun_out
bash scripts/dev/ab.sh c1_local c1
bash scripts/dev/ab.sh c1_chained c1 LINREC_LOCAL=0
bash scripts/dev/ab.sh c2 c2
timeout 600 python scripts/bench_kernel.py --out gpurun_out/bench_kernel.csv 2>&1 | grep -v Warn
LINREC_LOCAL=0 timeout 600 python scripts/bench_kernel.py --out gpurun_out/bench_kernel_chained.csv 2>&1 | grep -v Warn | grep "T="
