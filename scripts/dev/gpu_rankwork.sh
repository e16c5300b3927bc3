mkdir -p gpurun_out
for n in 2 4 8; do timeout 120 python scripts/rank_work.py $n 50 2>&1 | grep -v Warn; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/ncu_rankwork8.csv python scripts/rank_work.py 8 3 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/ncu_c4_launches.csv python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu --no-e2e --no-slow > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/ncu_c1_launches.csv python bench.py --workload c1 --steps 2 --warmup 1 --no-cpu --no-e2e --no-slow > /dev/null 2>&1
ls -la gpurun_out/*.csv
