# round-2 evidence: launch lists (our kernels only) for C2, C4, C1; ncu --set full of the C2 backward
# scan, the C4 forward fix-up and the C1 local scan; C3 layer bench (fp32 + tf32)
O=gpurun_out
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for wl in c2 c4 c1; do
  timeout 600 $NCU --metrics $M --clock-control none -k regex:"k_(tma|fixup|local|chain|vseg)" -c 24 --csv \
    --log-file $O/ncu_r02_launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 \
    > $O/ncu_r02_launches_$wl.log 2>&1; echo "$wl launches rc=$?"
done
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tma_bwd -s 2 -c 1 -o $O/ncu_r02_c2_bwd \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 > $O/ncu_r02_c2_bwd.log 2>&1; echo "c2 full rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_fixup -s 2 -c 2 -o $O/ncu_r02_c4_fixup \
  python bench.py --workload c4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow > $O/ncu_r02_c4_fixup.log 2>&1; echo "c4 full rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_local -s 4 -c 2 -o $O/ncu_r02_c1_local \
  python bench.py --workload c1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow > $O/ncu_r02_c1_local.log 2>&1; echo "c1 full rc=$?"
timeout 900 python bench.py --workload c3 --steps 10 --warmup 3 > $O/bench_r02_c3_fp32.json 2> $O/bench_r02_c3_fp32.err; echo "c3 rc=$?"
timeout 900 python bench.py --workload c3 --precision tf32 --steps 10 --warmup 3 > $O/bench_r02_c3_tf32.json 2> $O/bench_r02_c3_tf32.err; echo "c3 tf32 rc=$?"
ls -la $O | grep r02
