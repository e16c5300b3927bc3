for nt in 1 0 1 0; do
  LINREC_NT_COPY=$nt timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 --no-slow --no-extra 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('nt=$nt', round(e['value']/1e9,3), 'e9 el/s', round(e['ms_per_step'],1), 'ms; pinned', round(e['pinned']['value']/1e9,3))"
done
