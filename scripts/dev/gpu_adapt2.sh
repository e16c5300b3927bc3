timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/adapt_launches.csv python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-slow > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/adapt_launches.csv"))); hdr=None
out=[]
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); out.append((d["Kernel Name"].split("(")[0][:50], d["Grid Size"], d["Metric Value"]))
for x in out[-12:]: print(x)
PY
