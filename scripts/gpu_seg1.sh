O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_segments.py -q -m gpu --timeout 300 -p no:cacheprovider > $O/seg1_pytest.log 2>&1; echo "rc=$?" >> $O/seg1_pytest.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/seg1_pytest_all.log 2>&1; echo "rc=$?" >> $O/seg1_pytest_all.log
timeout 300 python bench.py --workload c4 --no-e2e --no-cpu > $O/seg1_bench_c4.log 2>&1; echo "rc=$?" >> $O/seg1_bench_c4.log
tail -n 30 $O/seg1_pytest.log | cut -c1-300; tail -n 3 $O/seg1_pytest_all.log; cut -c1-900 $O/seg1_bench_c4.log
