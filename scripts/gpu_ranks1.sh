O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_ranks.py tests/test_gpu_segments.py -q -m gpu --timeout 400 -p no:cacheprovider > $O/rk1_pytest.log 2>&1; echo "rc=$?" >> $O/rk1_pytest.log
LINREC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload c4 --steps 10 --warmup 3 > $O/rk1_bench_c4x2.log 2>&1; echo "rc=$?" >> $O/rk1_bench_c4x2.log
LINREC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu --e2e-steps 1 > $O/rk1_bench_c2x2.log 2>&1; echo "rc=$?" >> $O/rk1_bench_c2x2.log
LINREC_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/rk1_bench_refx2.log 2>&1; echo "rc=$?" >> $O/rk1_bench_refx2.log
tail -n 5 $O/rk1_pytest.log; for f in $O/rk1_bench_*.log; do echo "== $f"; tail -n 3 $f | cut -c1-700; done
