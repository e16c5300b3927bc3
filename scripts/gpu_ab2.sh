O=gpurun_out
export TUNE_FWD="12,2,8;16,1,8"
export TUNE_BWD="12,1,8;16,1,8"
for L in liblinrec_cuda.so scripts/ablib/liblinrec_cuda_t5.so; do
  for shape in "65536 8 1024" "1048576 1 128" "16777216 1 16"; do
    if [ $L = liblinrec_cuda.so ]; then LP=""; else LP=$L; fi
    LINREC_LIB_PATH=$LP timeout 200 python scripts/tune.py $shape >> $O/ab2.log 2>&1
  done
done
cat $O/ab2.log | python3 -c "
import sys,json
for l in sys.stdin:
  l=l.strip()
  try: d=json.loads(l)
  except Exception: print(l[:300]); continue
  print(d['lib'], d['T'], d['W'], d['kind'], d['fwd_cfg'], d['bwd_cfg'], 'fwd %.0f GB/s %.2f'%(d['fwd_gbs'],d['fwd_frac']) if 'fwd_gbs' in d else '', 'bwd %.0f GB/s %.2f'%(d['bwd_gbs'],d['bwd_frac']) if 'bwd_gbs' in d else '')
"
