timeout 900 python -m pytest tests/test_gpu_gated.py tests/test_gpu_layers.py tests/test_gpu_c3_fullsize.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null > gpurun_out/c3_gated.json
python -c "
import json; d=json.loads(open('gpurun_out/c3_gated.json').read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], {k: round(v['ms'],3) for k, v in d['stages'].items() if k in ('scan_bwd_cell','dc','h_out','scan_cell')})"
