mkdir -p gpurun_out
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "wall $(( $(date +%s) - t0 )) s"

python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_default.json").read().strip().splitlines()[-1])
print("C2", d["value"], d["ms_per_step"], d["roofline"]["frac"])
for k in ("c1", "c4", "c5", "c3"):
    v = d.get(k, {})
    print(k, v.get("value"), v.get("ms_per_step"), v.get("frac_of_peak_per_gpu"), (v.get("roofline") or {}).get("frac"), v.get("worst_point"))
print("e2e", d["e2e"]["value"], "cpu", d["cpu_baseline"]["value"])
PY
