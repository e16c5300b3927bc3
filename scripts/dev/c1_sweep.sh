# C1 (T=4096, W=256) per-direction times for several chain targets.
for c in 2 8 16 32 64 128 256; do
  r=$(LINREC_CHAINS=$c timeout 120 python bench.py --workload c1 --no-cpu --no-e2e --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print(round(d['ms_per_step']*1000,1),round(k['fwd']['ms']*1000,1),round(k['bwd']['ms']*1000,1))")
  echo "chains=$c $r"
done
