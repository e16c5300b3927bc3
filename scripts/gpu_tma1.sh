O=gpurun_out
timeout 300 python scripts/tune.py > $O/t1_tune.log 2>&1; echo "tune rc=$?" >> $O/t1_tune.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > $O/t1_pytest.log 2>&1; echo "pytest rc=$?" >> $O/t1_pytest.log
timeout 600 python bench.py --no-e2e --no-cpu > $O/t1_bench.log 2>&1; echo "bench rc=$?" >> $O/t1_bench.log
for f in $O/t1_tune.log $O/t1_pytest.log $O/t1_bench.log; do echo "== $f"; tail -n 15 $f; done
