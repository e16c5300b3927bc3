#!/usr/bin/env python
"""The paper's Table 3 on the B200: train the two-layer GILR-LSTM on the
synthetic long-dependency task (training.hpp run_experiment) until five
consecutive perfect minibatches, or time a fixed number of iterations.

    python scripts/train_synthetic.py --seq-len 1024 --hidden 512 [--batch 32]
        [--lr 1e-3] [--max-iters 5000] [--kernel-only] [--precision fp32|tf32]

Prints one JSON record: converged, iterations, wall / kernel seconds and the
mean seconds per iteration (CUDA-synchronised).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_04057_b200 import training as TR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq-len", type=int, default=1024)
    ap.add_argument("--hidden", type=int, default=512)
    ap.add_argument("--input-dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--max-iters", type=int, default=5000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--gate-bias", type=float, default=1.0)
    ap.add_argument("--kernel-only", action="store_true")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "tf32"])
    a = ap.parse_args()
    cfg = TR.TrainConfig(seq_len=a.seq_len, hidden=a.hidden, input_dim=a.input_dim, batch=a.batch,
                         learning_rate=a.lr, max_iters=a.max_iters, seed=a.seed, gate_bias=a.gate_bias,
                         time_data_gen=not a.kernel_only, precision=a.precision)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = TR.run_experiment(cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    last = rep.trace[-1]
    print(json.dumps({
        "seq_len": a.seq_len, "hidden": a.hidden, "input_dim": a.input_dim, "batch": a.batch, "lr": a.lr, "gate_bias": a.gate_bias,
        "precision": a.precision, "converged": rep.converged, "diverged": rep.diverged,
        "iterations": rep.iterations, "wall_seconds": wall, "timed_seconds": rep.elapsed_seconds,
        "seconds_per_iteration": rep.elapsed_seconds / rep.iterations, "final_loss": last.loss,
        "final_accuracy": last.accuracy, "diagnostic": rep.diagnostic,
        "device": torch.cuda.get_device_name(0),
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 2**30,
    }), flush=True)


if __name__ == "__main__":
    main()
