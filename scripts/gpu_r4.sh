O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r4_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r4_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/r4_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r4_pytest.log
timeout 900 python bench.py > $O/r4_bench.log 2>&1; echo "bench rc=$?" >> $O/r4_bench.log
timeout 600 python bench.py --workload c4 --no-e2e > $O/r4_bench_c4.log 2>&1; echo "bench rc=$?" >> $O/r4_bench_c4.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/r4_bench_ref.log 2>&1; echo "ref rc=$?" >> $O/r4_bench_ref.log
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/r4_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 2 -o $O/r4_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/r4_full.log 2>&1; echo "full rc=$?"
for f in $O/r4_smoke.log $O/r4_pytest.log; do echo "== $f"; tail -n 2 $f; done
for f in $O/r4_bench.log $O/r4_bench_c4.log $O/r4_bench_ref.log; do echo "== $f"; cut -c1-400 $f; done
