"""Summarise an `ncu --set full` report and a launch-list CSV into profiles/.

    python scripts/ncu_summary.py gpurun_out/r3_full.ncu-rep gpurun_out/r3_launches.csv profiles/ r01

Writes profiles/ncu_full_<tag>.csv (raw page, selected metrics),
profiles/ncu_launches_<tag>.csv (copied), profiles/ncu_full_summary.json (the
per-launch dram bytes bench.py reports as roofline.traffic).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "smsp__inst_executed.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__average_warp_latency_issue_stalled_barrier.ratio",
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def main(rep, launches, outdir, tag, elements=65536 * 8192):
    raw = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    keep = [i for i, h in enumerate(hdr) if h in METRICS]
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"ncu_full_{tag}.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([hdr[i] for i in keep])
        w.writerow([units[i] for i in keep])
        for r in rows[2:]:
            w.writerow([r[i] for i in keep])
    summary = {"source": f"ncu --set full --clock-control none, {os.path.basename(rep)}", "tag": tag}
    for r in rows[2:]:
        d = {hdr[i]: r[i] for i in range(len(hdr))}
        u = {hdr[i]: units[i] for i in range(len(hdr))}
        name = d["Kernel Name"]
        kind = "bwd" if "bwd" in name else "fwd"
        rd = float(d["dram__bytes_read.sum"]) * UNIT.get(u["dram__bytes_read.sum"], 1.0)
        wr = float(d["dram__bytes_write.sum"]) * UNIT.get(u["dram__bytes_write.sum"], 1.0)
        alg = (20 if kind == "bwd" else 12) * elements
        summary[kind] = {
            "kernel": name, "duration_ms": float(d["gpu__time_duration.sum"]) * (1e-6 if u["gpu__time_duration.sum"] == "ns" else 1e-3 if u["gpu__time_duration.sum"] == "us" else 1.0),
            "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
            "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
            "elements_per_launch": elements,
            "dram_throughput_pct_of_peak": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
            "registers": int(float(d["launch__registers_per_thread"])), "grid": int(float(d["launch__grid_size"])),
        }
    with open(os.path.join(outdir, "ncu_full_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    if launches and os.path.exists(launches):
        shutil.copy(launches, os.path.join(outdir, f"ncu_launches_{tag}.csv"))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
