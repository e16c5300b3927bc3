python scripts/dev/slow_c4.py 4 | tail -2
LINREC_ADAPTIVE=0 python scripts/dev/slow_c4.py 3 | tail -1
bash scripts/dev/ab.sh c4 c4
bash scripts/dev/ab.sh c4_noadapt c4 LINREC_ADAPTIVE=0
bash scripts/dev/ab.sh c2 c2
bash scripts/dev/ab.sh c2_noadapt c2 LINREC_ADAPTIVE=0
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c4_fullsize.py tests/test_gpu_segments.py -x -q 2>&1 | tail -2
