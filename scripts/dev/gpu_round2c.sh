mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_c3_fullsize.py -x -q > gpurun_out/pytest_c3.log 2>&1
tail -15 gpurun_out/pytest_c3.log
python scripts/dev/host_copy_bw.py > gpurun_out/host_copy_bw.txt 2>&1
cat gpurun_out/host_copy_bw.txt
