# evidence for the cluster scans (C1) and refreshed bench lines on the current code:
# C1 launch list, a full capture of k_cluster_bwd, bench lines for C1 / C4 / the default C2
O=gpurun_out
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 $NCU --metrics $M --clock-control none -k regex:"k_" -c 30 --csv \
  --log-file $O/ncu_r02_cluster_launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 --no-extra \
  > /dev/null 2>&1; echo "c1 launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_cluster_bwd -s 2 -c 1 -o $O/ncu_r02_cluster_c1_bwd \
  python bench.py --workload c1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 --no-extra > /dev/null 2>&1; echo "c1 full rc=$?"
$NCU -i $O/ncu_r02_cluster_c1_bwd.ncu-rep --page raw --csv > $O/ncu_r02_full_c1_cluster_bwd.csv 2>/dev/null
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_cluster_fwd -s 2 -c 1 -o $O/ncu_r02_cluster_c1_fwd \
  python bench.py --workload c1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-slow --no-c4 --no-extra > /dev/null 2>&1; echo "c1 fwd full rc=$?"
$NCU -i $O/ncu_r02_cluster_c1_fwd.ncu-rep --page raw --csv > $O/ncu_r02_full_c1_cluster_fwd.csv 2>/dev/null
timeout 600 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo "c1 bench rc=$?"
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "default bench rc=$?"
