# usage: bash scripts/gpu_prof.sh TAG -- launch list + ncu --set full of the chained kernels
TAG=${1:-prof}
O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_launches_bench.log 2>&1
echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_chain -s 4 -c 2 -o $O/${TAG}_full \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/${TAG}_full.log 2>&1
echo "full rc=$?"
ls -la $O/ | grep $TAG
