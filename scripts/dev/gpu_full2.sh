mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1
tail -5 gpurun_out/pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; tail -c 300 gpurun_out/bench_c1.json
