O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/vs2_pytest.log 2>&1; echo "rc=$?" >> $O/vs2_pytest.log
export TUNE_FWD="12,2,8"
export TUNE_BWD="12,1,8"
TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py > $O/vs2_tune.log 2>&1
TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py 1048576 1 128 >> $O/vs2_tune.log 2>&1
TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py 16777216 1 16 >> $O/vs2_tune.log 2>&1
TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py 4096 1 256 >> $O/vs2_tune.log 2>&1
grep -E "passed|failed|Error|error" $O/vs2_pytest.log | tail -15
cat $O/vs2_tune.log | python3 -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  try: d=json.loads(l)
  except Exception: print(l[:300]); continue
  print(d['T'], d['W'], d['kind'], d['fwd_cfg'], d['bwd_cfg'], 'fwd %.0f GB/s %.2f'%(d['fwd_gbs'],d['fwd_frac']) if 'fwd_gbs' in d else '', 'bwd %.0f GB/s %.2f'%(d['bwd_gbs'],d['bwd_frac']) if 'bwd_gbs' in d else '', 'err %.1e'%max(d.get('fwd_err',0),d.get('bwd_err',0)))
"
