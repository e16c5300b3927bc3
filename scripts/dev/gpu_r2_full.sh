# round 2 re-entry: full GPU suite + default bench + C4/C5 records
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1
tail -15 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
tail -c 1500 gpurun_out/bench_default.err
timeout 600 python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 1000 gpurun_out/bench_c5.err
