python scripts/dev/slow_c4.py 4 | tail -2
bash scripts/dev/ab.sh c4 c4
bash scripts/dev/ab.sh c2 c2
timeout 900 python -m pytest tests/test_gpu_segments.py tests/test_gpu_c4_fullsize.py tests/test_gpu_parity.py tests/test_gpu_sharded_ranks.py -x -q 2>&1 | tail -2
