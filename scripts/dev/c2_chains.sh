# C2 forward vs. the forward chain target (64: no virtual segments, no fix-up).
for c in 64 128 256 512; do
  r=$(LINREC_CHAINS_FWD=$c timeout 200 python bench.py --no-cpu --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print(round(d['ms_per_step']*1000,1),round(k['fwd']['ms']*1000,1),round(k['bwd']['ms']*1000,1))")
  echo "fwd_chains=$c $r"
done
