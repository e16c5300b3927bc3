# Stitch-path check on one B200: segment / parity / sharded tests, C4 bench,
# per-rank N=8 work and its launch list.  Results in gpurun_out/.
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_segments.py tests/test_gpu_parity.py tests/test_gpu_sharded_ranks.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do
  timeout 120 python bench.py --workload c4 --no-cpu --no-e2e > $O/c4.json
  python -c "import json;d=json.load(open('$O/c4.json'));print('c4',d['value'],d['ms_per_step'],d['kernels']['fwd']['ms'],d['kernels']['bwd']['ms'])"
done
python scripts/rank_work.py 8 | tail -2
timeout 300 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum -c 40 --csv \
  --log-file $O/rank8.csv python scripts/rank_work.py 8 3 >/dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.DictReader(l for l in open('gpurun_out/rank8.csv') if not l.startswith('==')) if r.get('Metric Name')=='gpu__time_duration.sum']
for r in rows[-11:]:
    print(round(float(r['Metric Value'])/1000,1), r['Grid Size'], r['Kernel Name'][:60])
PY
