O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r3_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r3_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/r3_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r3_pytest.log
timeout 900 python bench.py > $O/r3_bench.log 2>&1; echo "bench rc=$?" >> $O/r3_bench.log
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/r3_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/r3_launches_bench.log 2>&1; echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 2 -o $O/r3_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/r3_full.log 2>&1; echo "full rc=$?"
for f in $O/r3_smoke.log $O/r3_pytest.log $O/r3_bench.log; do echo "== $f"; tail -n 3 $f | cut -c1-600; done
