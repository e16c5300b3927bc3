for tf in 1 0; do
LINREC_TAIL_FOLD=$tf timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 30 --csv --log-file gpurun_out/tail_$tf.csv python scripts/rank_work.py 8 2 > /dev/null 2>&1
python - $tf <<'PY'
import csv, sys
rows=list(csv.reader(open(f"gpurun_out/tail_{sys.argv[1]}.csv"))); hdr=None; out=[]
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.append((d["Kernel Name"].split("(")[0][:40], d["Grid Size"], d["Metric Value"]))
print("tail_fold", sys.argv[1]); [print("  ",x) for x in out[-8:]]
PY
done
