for c in 48 64 96 128; do
  r=$(LINREC_CHAINS_BWD=$c timeout 200 python bench.py --workload c4 --no-cpu --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print(round(d['ms_per_step']*1000,1),round(k['fwd']['ms']*1000,1),round(k['bwd']['ms']*1000,1))")
  echo "bwd_chains=$c $r"
done
