O=gpurun_out
export TUNE_FWD="12,2,8;16,1,8"
export TUNE_BWD="12,1,8;16,1,8"
for i in 1 2; do
timeout 200 python scripts/tune.py >> $O/ab1_new.log 2>&1
LINREC_LIB_PATH=scripts/ablib/liblinrec_cuda_t3.so timeout 200 python scripts/tune.py >> $O/ab1_old.log 2>&1
done
for f in $O/ab1_new.log $O/ab1_old.log; do echo "== $f"; cat $f | python3 -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  try: d=json.loads(l)
  except Exception: print(l[:300]); continue
  print(d['lib'], d.get('sm_mhz'), d['kind'], d['fwd_cfg'], d['bwd_cfg'], 'fwd %.0f GB/s %.2f'%(d['fwd_gbs'],d['fwd_frac']) if 'fwd_gbs' in d else '', 'bwd %.0f GB/s %.2f'%(d['bwd_gbs'],d['bwd_frac']) if 'bwd_gbs' in d else '')
"; done
