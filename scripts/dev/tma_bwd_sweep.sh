for cfg in "12,1,8" "8,2,8" "10,1,8" "16,1,8"; do
  for w in c4 c2; do
    r=$(LINREC_TMA_BWD=$cfg timeout 200 python bench.py --workload $w --no-cpu --no-e2e --steps 30 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print(round(d['ms_per_step']*1000,1),round(k['bwd']['ms']*1000,1))")
    echo "bwd=$cfg $w $r"
  done
done
