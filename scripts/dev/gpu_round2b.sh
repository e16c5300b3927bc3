# round 2: new GPU tests (check_finite, shape contract, C++ sharded ranks) + staged e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cpp_api.py tests/test_gpu_parity.py -x -q -k "cpp or finite or shape_contract or numpy or host" > gpurun_out/pytest_b.log 2>&1
tail -15 gpurun_out/pytest_b.log
python bench.py --steps 5 --no-cpu --no-c4 --no-slow > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
tail -c 1500 gpurun_out/bench_e2e.json
