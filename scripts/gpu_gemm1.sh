O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu --timeout 120 -p no:cacheprovider -x > $O/gm1_pytest.log 2>&1; echo "rc=$?" >> $O/gm1_pytest.log
tail -n 30 $O/gm1_pytest.log | cut -c1-300
