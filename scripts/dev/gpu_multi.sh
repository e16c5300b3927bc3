mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"
python scripts/dev/host_copy_bw.py 2>&1 | tail -8
LINREC_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err
tail -c 2500 gpurun_out/bench_g2.json; grep -v "Warn\|warn_once" gpurun_out/bench_g2.err | tail -5
