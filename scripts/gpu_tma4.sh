O=gpurun_out
export TUNE_FWD="12,2,8;10,2,8;8,2,8;16,1,8;12,1,8"
export TUNE_BWD="12,1,8;10,1,8;8,2,8;16,1,8"
timeout 300 python scripts/tune.py > $O/t4_tune.log 2>&1; echo "tune rc=$?" >> $O/t4_tune.log
export TUNE_FWD="12,2,8;8,2,8"
export TUNE_BWD="12,1,8;8,2,8"
timeout 300 python scripts/tune.py 1048576 1 128 > $O/t4_tune_c4.log 2>&1; echo "tune rc=$?" >> $O/t4_tune_c4.log
timeout 300 python scripts/tune.py 4096 1 256 > $O/t4_tune_c1.log 2>&1; echo "tune rc=$?" >> $O/t4_tune_c1.log
timeout 300 python scripts/tune.py 16777216 1 16 > $O/t4_tune_c5.log 2>&1; echo "tune rc=$?" >> $O/t4_tune_c5.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider -x > $O/t4_pytest.log 2>&1; echo "pytest rc=$?" >> $O/t4_pytest.log
for f in $O/t4_tune.log $O/t4_tune_c4.log $O/t4_tune_c1.log $O/t4_tune_c5.log $O/t4_pytest.log; do echo "== $f"; cat $f | python3 -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  try: d=json.loads(l)
  except Exception: print(l[:300]); continue
  print(d['kind'], d['fwd_cfg'], d['bwd_cfg'], 'fwd %.0f GB/s %.2f'%(d['fwd_gbs'],d['fwd_frac']) if 'fwd_gbs' in d else '', 'bwd %.0f GB/s %.2f'%(d['bwd_gbs'],d['bwd_frac']) if 'bwd_gbs' in d else '', 'err %.1e'%max(d.get('fwd_err',0),d.get('bwd_err',0)))
"; done
