#!/usr/bin/env python
"""GPU mirror of the reference's kernel benchmark (bench.hpp:160-244
bench_kernel; the paper's Table 1): the serial scan vs the
parallel scan on identical inputs at every (T, n, b) grid point, forward only.

Protocol, as the reference's:
  * inputs per grid point idx from Rng(seed).split(1000 + idx):
    lam ~ U(0.05, 0.95), x, h0 ~ U(-1, 1) (bench.hpp:134-143, 186), drawn on the
    host with the repo's restatement of rng.hpp (training.Rng), checksummed with
    FNV-1a 64 exactly as checksum_inputs (bench.hpp:69-85) -- so every row can
    be matched to the reference's own row on the same inputs;
  * `warmup` untimed calls, then the MEDIAN of `reps` timed calls
    (median_rep_seconds, bench.hpp:93-107); here a rep is one replay of a
    CUDA graph of 20 back-to-back launches timed with CUDA events (inputs
    resident in HBM), divided by 20 -- the GPU time per launch;
  * correctness guard: parallel vs serial within 2e-4 x max(|h_serial|, 1)
    (bench.hpp:203-213), else the run fails;
  * events/s = b * T * reps / (median * reps); speedup = serial / parallel;
  * CSV: `# ` metadata lines, then "T,n,b,workers,impl,events_per_sec,speedup"
    (write_bench_csv, bench.hpp:418-432).  `workers` is the SM count (the
    GPU's "pool"); an extra column-free metadata line records the checksums.

Serial = the per-channel kernel (mode "serial", bit-exact to the reference);
parallel = the library's parallel mode (the CTA-local scan for T <= 4096 and
<= 2^21 elements, the chained look-back scan otherwise).

Usage: python scripts/bench_kernel.py [--seq-lens 16,256,4096,65536]
       [--features 4,32,128] [--batches 1] [--warmup 3] [--reps 10]
       [--seed 0] [--out profiles/bench_kernel_r02.csv]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402
from paper_1709_04057_b200.training import Rng  # noqa: E402

PAPER_TABLE1 = {  # PAPER.md:328-336 (K80, m features, b = 1): parallel / serial speedup
    (16, 4): 0.06, (16, 32): 0.06, (16, 128): 0.05,
    (256, 4): 0.22, (256, 32): 0.22, (256, 128): 0.86,
    (4096, 4): 1.02, (4096, 32): 2.94, (4096, 128): 3.36,
    (65536, 4): 38.5, (65536, 32): 41.8, (65536, 128): 17.5,
}


def ints(s):
    return [int(v) for v in s.split(",") if v]


def inputs(seed, idx, T, b, n):
    rng = Rng(seed).split(1000 + idx)
    lam = rng.uniform_array(T * b * n, 0.05, 0.95).astype(np.float32).reshape(T, b, n)
    x = rng.uniform_array(T * b * n, -1.0, 1.0).astype(np.float32).reshape(T, b, n)
    h0 = rng.uniform_array(b * n, -1.0, 1.0).astype(np.float32).reshape(b, n)
    return lam, x, h0


def median_rep_us(fn, warmup, reps, stream, per_graph=20):
    """Median over `reps` of the per-launch GPU time: each rep replays a CUDA
    graph of `per_graph` back-to-back launches (so host launch overhead, ~10 us
    through Python, does not masquerade as kernel time at small T)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(per_graph):
            fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    with torch.cuda.stream(stream):  # replay() launches on the current stream
        g.replay()
        torch.cuda.synchronize()
        for r in range(reps):
            ev[2 * r].record(stream)
            g.replay()
            ev[2 * r + 1].record(stream)
    torch.cuda.synchronize()
    return statistics.median(ev[2 * r].elapsed_time(ev[2 * r + 1]) * 1e3 / per_graph for r in range(reps))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-lens", default="16,256,4096,65536")
    ap.add_argument("--features", default="4,32,128")
    ap.add_argument("--batches", default="1")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "bench_kernel_r02.csv"))
    args = ap.parse_args(argv)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    stream = torch.cuda.Stream(device=dev)
    st = stream.cuda_stream
    ws = capi.Workspace(0)  # explicit look-back workspace: graph-capturable
    rows, md, sums = [], [], []
    point = 0
    for T in ints(args.seq_lens):
        for n in ints(args.features):
            for b in ints(args.batches):
                idx = point
                point += 1
                lam, x, h0 = inputs(args.seed, idx, T, b, n)
                csum = capi.fnv1a64(lam, x, h0)
                L, X, H0 = (torch.from_numpy(a).to(dev) for a in (lam, x, h0))
                hs, hp = torch.empty_like(L), torch.empty_like(L)
                W = b * n
                ser = median_rep_us(lambda: capi.scan(L.data_ptr(), X.data_ptr(), H0.data_ptr(), hs.data_ptr(), T, W,
                                                      capi.SERIAL, 4, ws.handle, st), args.warmup, args.reps, stream)
                par = median_rep_us(lambda: capi.scan(L.data_ptr(), X.data_ptr(), H0.data_ptr(), hp.data_ptr(), T, W,
                                                      capi.PARALLEL, 4, ws.handle, st), args.warmup, args.reps, stream)
                a, r = hp.double(), hs.double()
                worst = (a - r).abs().max().item()
                scale = max(r.abs().max().item(), 1.0)
                if worst > 2e-4 * scale:
                    raise SystemExit(f"bench_kernel: serial/parallel disagreement at T={T} n={n} b={b}")
                events = b * T
                rows.append((T, n, b, sms, "serial", events / (ser * 1e-6), 1.0, ser))
                rows.append((T, n, b, sms, "parallel", events / (par * 1e-6), ser / par, par))
                sums.append((T, n, b, csum))
                print(f"T={T:6d} n={n:4d} b={b}: serial {ser:9.1f} us  parallel {par:8.1f} us  "
                      f"speedup {ser / par:7.2f}  (paper K80: {PAPER_TABLE1.get((T, n), '-')})  "
                      f"fnv1a64 {csum:016x}", flush=True)
    md.append(f"bench_kernel (bench.hpp:160-244) on {torch.cuda.get_device_name(dev)}, {sms} SMs, fp32, forward")
    md.append(f"seed={args.seed} warmup={args.warmup} reps={args.reps} (median of reps; a rep = one CUDA-graph replay "
              f"of 20 back-to-back launches, time / 20)")
    md.append("workers = SM count; serial = per-channel kernel, parallel = linrec parallel mode")
    for T, n, b, c in sums:
        md.append(f"input_checksum T={T} n={n} b={b}: {c:016x}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        for line in md:
            f.write(f"# {line}\n")
        f.write("T,n,b,workers,impl,events_per_sec,speedup\n")
        for T, n, b, w, impl, eps, sp, _ in rows:
            f.write(f"{T},{n},{b},{w},{impl},{eps:.9g},{sp:.9g}\n")
    print(f"wrote {args.out}")
    return rows, sums


if __name__ == "__main__":
    main()
