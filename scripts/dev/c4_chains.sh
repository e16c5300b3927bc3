for cb in 64 128 256; do for cf in 256 512; do
  r=$(LINREC_CHAINS_FWD=$cf LINREC_CHAINS_BWD=$cb timeout 120 python bench.py --workload c4 --no-cpu --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print(round(d['ms_per_step']*1000,1),round(k['fwd']['ms']*1000,1),round(k['bwd']['ms']*1000,1))")
  echo "fwd=$cf bwd=$cb $r"
done; done
