#!/bin/bash
# Round-end evidence run on one B200 (through gpurun); everything lands in
# gpurun_out/ and is summarised into profiles/ by scripts/ncu_summary.py.
set -x
O=gpurun_out
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_c2_reference.json 2>> $O/bench.err
timeout 600 python bench.py --workload c4 --no-cpu > $O/bench_c4.json 2>> $O/bench.err
timeout 600 python bench.py --workload c3 > $O/bench_c3_fp32.json 2>> $O/bench.err
timeout 600 python bench.py --workload c3 --precision tf32 --no-cpu --no-e2e > $O/bench_c3_tf32.json 2>> $O/bench.err
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
  python bench.py --workload c4 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c3.csv \
  python bench.py --workload c3 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tma -s 4 -c 2 -o $O/full_c2 -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/full_c2.log 2>&1
timeout 900 python scripts/bench_model.py --out $O/bench_model_r01.json > $O/bench_model.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
