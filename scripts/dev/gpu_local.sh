mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_channel_sharded.py -x -q > gpurun_out/pytest_local.log 2>&1; tail -3 gpurun_out/pytest_local.log
bash scripts/dev/ab.sh c1_local c1
bash scripts/dev/ab.sh c1_chained c1 LINREC_LOCAL=0
timeout 600 python scripts/bench_kernel.py --out gpurun_out/bench_kernel.csv 2>&1 | grep -v Warn
LINREC_LOCAL=0 timeout 600 python scripts/bench_kernel.py --out gpurun_out/bench_kernel_chained.csv 2>&1 | grep -v Warn
