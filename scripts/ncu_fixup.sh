# Launch lists of the C4 stitch kernels for several fix-up walker counts.
O=gpurun_out
for w in 1 2 4; do
  LINREC_FIXUP_WALK=$w timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
    -c 40 --csv --log-file $O/fixup_walk$w.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-e2e --no-cpu >/dev/null 2>&1
done
