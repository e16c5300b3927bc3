# final round-2 evidence on the final code: launch lists (our kernels) for C2 / C4 / C1 / C3,
# full capture of the C2 backward scan, the default bench line, the GPU test suite
O=gpurun_out
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for wl in c2 c4 c1; do
  timeout 600 $NCU --metrics $M --clock-control none -k regex:"k_" -c 30 --csv \
    --log-file $O/ncu_r02_final_launches_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 --no-extra \
    > /dev/null 2>&1; echo "$wl launches rc=$?"
done
timeout 900 $NCU --metrics $M --clock-control none -k regex:"k_" -c 60 --csv --log-file $O/ncu_r02_final_launches_c3.csv \
  python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "c3 launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tma_bwd -s 2 -c 1 -o $O/ncu_r02_final_c2_bwd \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 --no-extra > /dev/null 2>&1; echo "c2 full rc=$?"
