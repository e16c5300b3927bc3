mkdir -p gpurun_out
python bench.py --steps 5 --no-cpu --no-c4 --no-slow > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "import json;d=json.loads(open('gpurun_out/bench_e2e.json').read().splitlines()[-1]);print(d['value'],d['e2e'])"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1
tail -15 gpurun_out/pytest_full.log
