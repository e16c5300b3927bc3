#!/usr/bin/env python
"""Whole-model throughput on the B200: the reference's ``bench_model``
(proj/include/linrec/bench.hpp:246-414) -- the regime of the paper's Table 2.

Two stacked layers of ``arch`` (gilr, gilr-lstm, qrnn-k2, qrnn-k10) at the
reference preset (input m = 4, hidden n = 256, b*T = 65536 held constant
across the sequence-length grid, bench.hpp:28-31), one train-shaped step =
forward + backward of both layers with d_h = 1 (bench.hpp:281-310).  Each grid
point is timed with the recurrences on the per-channel serial kernel
(ScanMode::Serial) and on the chained parallel scans, alternating the two
(median_paired_seconds, bench.hpp:367-373), with the reference's guard
(serial vs parallel h within 2e-4 normwise, bench.hpp:375-384).  Everything
else -- the tcgen05 gate GEMMs, the pointwise kernels -- is identical in both
columns, exactly as in the reference where only the ThreadPool/ScanMode
changes.

    python scripts/bench_model.py [--archs ...] [--seq-lens ...] [--reps 10]
        [--precision fp32|tf32] [--out profiles/bench_model_r01.json]

Times are CUDA events on the launching stream (device time of the whole
step); events/s = b*T / step time (bench.hpp:386).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1709_04057_b200 import layers as L  # noqa: E402


class Model:
    """detail::ModelUnderBench (bench.hpp:251-311) on the GPU."""

    def __init__(self, arch, m, n, gen, precision):
        self.arch, self.n, self.prec = arch, n, precision
        if arch == "gilr":
            self.p = [L.gilr_init(gen, m, n, 1.0), L.gilr_init(gen, n, n, 1.0)]
        elif arch == "gilr-lstm":
            self.p = [L.gilr_lstm_init(gen, m, n, 1.0), L.gilr_lstm_init(gen, n, n, 1.0)]
        elif arch in ("qrnn-k2", "qrnn-k10"):
            k = 2 if arch == "qrnn-k2" else 10
            self.p = [L.qrnn_init(gen, m, n, k, 1.0), L.qrnn_init(gen, n, n, k, 1.0)]
        else:
            raise ValueError(f'bench_model: unknown arch "{arch}"')

    def step(self, x, zero, mode):
        T, b, _ = x.shape
        d_h = torch.ones(T, b, self.n, device=x.device)
        kw = dict(mode=mode, precision=self.prec)
        if self.arch == "gilr":
            c1, c2 = L.GilrCache(), L.GilrCache()
            h1 = L.gilr_forward(self.p[0], x, zero, cache=c1, **kw)
            h2 = L.gilr_forward(self.p[1], h1, zero, cache=c2, **kw)
            g1, g2 = L.GilrGrads.zeros_like(self.p[0]), L.GilrGrads.zeros_like(self.p[1])
            d1, _ = L.gilr_backward(self.p[1], h1, zero, c2, d_h, g2, **kw)
            L.gilr_backward(self.p[0], x, zero, c1, d1, g1, **kw)
            return h2
        if self.arch == "gilr-lstm":
            c1, c2 = L.GilrLstmCache(), L.GilrLstmCache()
            h1 = L.gilr_lstm_forward(self.p[0], x, zero, zero, cache=c1, **kw)
            h2 = L.gilr_lstm_forward(self.p[1], h1, zero, zero, cache=c2, **kw)
            g1, g2 = L.GilrLstmGrads.zeros_like(self.p[0]), L.GilrLstmGrads.zeros_like(self.p[1])
            d1, _, _ = L.gilr_lstm_backward(self.p[1], h1, zero, zero, c2, d_h, g2, **kw)
            L.gilr_lstm_backward(self.p[0], x, zero, zero, c1, d1, g1, **kw)
            return h2
        c1, c2 = L.QrnnCache(), L.QrnnCache()
        h1 = L.qrnn_forward(self.p[0], x, zero, cache=c1, **kw)
        h2 = L.qrnn_forward(self.p[1], h1, zero, cache=c2, **kw)
        g1, g2 = L.QrnnGrads.zeros_like(self.p[0]), L.QrnnGrads.zeros_like(self.p[1])
        d1, _ = L.qrnn_backward(self.p[1], h1, zero, c2, d_h, g2, **kw)
        L.qrnn_backward(self.p[0], x, zero, c1, d1, g1, **kw)
        return h2


def timed(fn, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    out = fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / 1e3, out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--archs", nargs="+", default=["gilr", "gilr-lstm", "qrnn-k2", "qrnn-k10"])
    ap.add_argument("--seq-lens", nargs="+", type=int, default=[16, 256, 4096, 65536])
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--input", type=int, default=4)
    ap.add_argument("--bt", type=int, default=65536)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    records = []
    for arch in args.archs:
        for T in args.seq_lens:
            if args.bt % T:
                records.append({"arch": arch, "T": T, "skipped": True, "warning": "preset bT is not divisible by T"})
                continue
            b = args.bt // T
            k = 10 if arch == "qrnn-k10" else 2
            if arch.startswith("qrnn") and k > T:
                records.append({"arch": arch, "T": T, "skipped": True,
                                "warning": "filter window exceeds sequence length"})
                continue
            gen = torch.Generator().manual_seed(2000 + len(records))
            model = Model(arch, args.input, args.hidden, gen, args.precision)
            x = (torch.rand(T, b, args.input, generator=gen) * 2 - 1).to(dev)
            zero = torch.zeros(b, args.hidden, device=dev)
            ser, par = [], []
            h_s = h_p = None
            for i in range(args.warmup + args.reps):  # alternate the two modes
                ts, h_s = timed(lambda: model.step(x, zero, "serial"), stream)
                tp, h_p = timed(lambda: model.step(x, zero, "parallel"), stream)
                if i >= args.warmup:
                    ser.append(ts)
                    par.append(tp)
            worst = (h_s - h_p).abs().max().item()
            scale = max(h_s.abs().max().item(), 1.0)
            if worst > 2e-4 * scale:
                raise SystemExit(f"bench_model: serial/parallel disagreement at T={T} ({worst:.3e})")
            s, p = statistics.median(ser), statistics.median(par)
            rec = {"arch": arch, "T": T, "b": b, "n": args.hidden, "m": args.input, "reps": args.reps,
                   "precision": args.precision,
                   "serial": {"seconds": s, "events_per_sec": b * T / s},
                   "parallel": {"seconds": p, "events_per_sec": b * T / p},
                   "speedup": s / p, "guard_max_abs_diff": worst}
            records.append(rec)
            print(json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"device": torch.cuda.get_device_name(dev), "preset": vars(args), "records": records}, f,
                      indent=1)
        md = os.path.splitext(args.out)[0] + ".md"
        with open(md, "w") as f:
            f.write(f"# bench_model on {torch.cuda.get_device_name(dev)} (2 layers, m={args.input}, "
                    f"n={args.hidden}, bT={args.bt}, {args.precision})\n\n")
            f.write("| arch | T | b | serial events/s | parallel events/s | speedup |\n|---|---|---|---|---|---|\n")
            for r in records:
                if r.get("skipped"):
                    f.write(f"| {r['arch']} | {r['T']} | - | skipped: {r['warning']} | | |\n")
                else:
                    f.write(f"| {r['arch']} | {r['T']} | {r['b']} | {r['serial']['events_per_sec']:.3e} | "
                            f"{r['parallel']['events_per_sec']:.3e} | {r['speedup']:.2f} |\n")
    return records


if __name__ == "__main__":
    main()
