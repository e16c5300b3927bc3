set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_gpu.txt 2>&1
(nproc; lscpu | grep -E "Model name|Socket|Thread|Core") > gpurun_out/r1_host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 600 python bench.py > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r1_bench.log
tail -3 gpurun_out/r1_smoke.log gpurun_out/r1_pytest.log gpurun_out/r1_bench.log
