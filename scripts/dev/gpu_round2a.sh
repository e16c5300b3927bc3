set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -c 3000 gpurun_out/bench_c2.err
python bench.py --workload c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 2000 gpurun_out/bench_c5.err
timeout 900 python -m pytest tests/test_gpu_c4_fullsize.py tests/test_gpu_sharded_ranks.py -x -q > gpurun_out/pytest_new.log 2>&1
tail -30 gpurun_out/pytest_new.log
