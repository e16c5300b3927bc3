M=gpu__time_duration.sum
LINREC_ADAPTIVE=0 timeout 300 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:"k_" --csv --log-file gpurun_out/n8_plain.csv python scripts/dev/plain_scan.py 131072 128 > /dev/null 2>&1
timeout 300 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:"k_" -c 24 --csv --log-file gpurun_out/n8_seg.csv python scripts/rank_work.py 8 2 > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/n8_plain.csv", "gpurun_out/n8_seg.csv"):
    rows=list(csv.reader(open(f))); hdr=None; out=[]
    for r in rows:
        if r and r[0]=="ID": hdr=r; continue
        if hdr and len(r)==len(hdr):
            d=dict(zip(hdr,r)); out.append((d["Kernel Name"].split("(")[0][:45], d["Grid Size"], d["Metric Value"]))
    print(f); [print("  ",x) for x in out[-8:]]
PY
