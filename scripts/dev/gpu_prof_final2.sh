# launch lists of the final code for C2 / C4 / C1 (bench decays and, for C2 / C4, the
# slow-decay record: the decay-adaptive stitch's deep branches)
O=gpurun_out
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for wl in c2 c4 c1; do
  timeout 900 $NCU --metrics $M --clock-control none -k regex:"k_" -c 200 --csv \
    --log-file $O/ncu_r02_final2_launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-e2e --no-cpu --no-c4 --no-extra \
    > /dev/null 2>&1; echo "$wl launches rc=$?"
done
