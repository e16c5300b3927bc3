# A/B helper: bash scripts/dev/ab.sh LABEL WORKLOAD [ENV=VAL ...]  -> one line of fwd/bwd us (+ slow decay)
lab=$1; wl=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e --no-c4 > gpurun_out/ab_$lab.json 2> gpurun_out/ab_$lab.err
python - "$lab" <<'PY' || tail -5 gpurun_out/ab_$lab.err
import json, sys
lab = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{lab}.json").read().strip().splitlines()[-1])
s = d.get("slow_decay", {})
print("%-22s %.3e el/s  fwd %7.1f us  bwd %7.1f us  guard %.1e | slow %.3e fwd %7.1f bwd %7.1f" % (
    lab, d["value"], 1e3*d["kernels"]["fwd"]["ms"], 1e3*d["kernels"]["bwd"]["ms"], d["config"]["guard_max_rel_err"],
    s.get("value", 0), 1e3*s.get("fwd_ms", 0), 1e3*s.get("bwd_ms", 0)))
PY
