O=gpurun_out
timeout 300 python scripts/tune.py > $O/t3_tune.log 2>&1; echo "tune rc=$?" >> $O/t3_tune.log
timeout 300 python scripts/tune.py 1048576 1 128 > $O/t3_tune_c4.log 2>&1; echo "tune rc=$?" >> $O/t3_tune_c4.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_tma -s 4 -c 2 -o $O/t3_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/t3_full.log 2>&1; echo "ncu rc=$?"
for f in $O/t3_tune.log $O/t3_tune_c4.log; do echo "== $f"; cat $f | cut -c1-330; done
