O=gpurun_out
export TUNE_FWD="12,2,8"
export TUNE_BWD="12,1,8"
for CH in 64 128 256; do
for shape in "65536 8 1024" "1048576 1 128" "16777216 1 16" "4096 1 256"; do
  LINREC_CHAINS=$CH TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py $shape 2>/dev/null | sed "s/^/{\"chains\": $CH, \"r\": /; s/}$/}}/" >> $O/vs3_tune.log
done; done
LINREC_NARROW_COLUMNS=1 TUNE_NO_REGISTER=1 timeout 200 python scripts/tune.py 1048576 1 128 2>/dev/null | sed "s/^/{\"chains\": \"narrow\", \"r\": /; s/}$/}}/" >> $O/vs3_tune.log
cat $O/vs3_tune.log | python3 -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  try: o=json.loads(l); d=o['r']
  except Exception: print(l[:200]); continue
  print(o['chains'], d['T'], d['W'], d['fwd_cfg'], d['bwd_cfg'], 'fwd %.0f GB/s %.2f'%(d['fwd_gbs'],d['fwd_frac']) if 'fwd_gbs' in d else '', 'bwd %.0f GB/s %.2f'%(d['bwd_gbs'],d['bwd_frac']) if 'bwd_gbs' in d else '', 'err %.1e'%max(d.get('fwd_err',0),d.get('bwd_err',0)))
"
