#!/usr/bin/env python
"""Benchmark of the linear-recurrence hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c4|c1|c3] [--precision fp32|tf32]

One step = one forward scan (lam, x, h0 -> h) + one reverse-time backward scan
(lam, h0, h, dh -> dlam, dx, dh0) over one batch of synthetic input, fp32.
Default workload = BASELINE configs[1] ("C2"): T=65536, B=8, D=1024 on 1 GPU.

* ``value``      elements/s fwd+bwd (N_elements / step time), inputs resident in
                 HBM, device-timed with CUDA events on the launching stream, max
                 over ranks; each tensor is 2 GiB >> the 126 MB L2, so no flush
                 is needed between steps.
* ``e2e``        the same metric through the numpy-facing C ABI host entry points
                 (linrec_scan_host_f32 / linrec_scan_backward_host_f32) from
                 pinned host buffers: H2D of the inputs and D2H of every output
                 inside the timed region.
* ``roofline``   dominant kernel (the backward scan: 20 of the 32 algorithmic
                 B/element) -- algorithmic bytes / measured launch time vs the
                 measured HBM copy peak (MEASURED_PEAKS.json).
* ``cpu_baseline`` the reference's own CPU path (oracle/_ref, compiled from
                 /root/reference) on this host's cores, bounded sample.

Multi-GPU (torchrun, one rank per GPU): workload c2 is channel-sharded (each
rank owns an independent [T, W] block, no data-path collective; weak scaling);
workload c4 (T = 2^20, W = 128) is sequence-sharded with one carry all-gather
per direction (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import re
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan elements/s fwd+bwd and HBM GB/s (% of peak) at 1/2/4/8 B200 vs host CPU"
FWD_BYTES = 12  # fp32 algorithmic bytes per element: read lam, x; write h
BWD_BYTES = 20  # read lam, h, dh; write dlam, dx
WORKLOADS = {
    "c1": dict(T=4096, B=1, D=256, desc="C1 fp32 linear recurrence T=4096 B=1 D=256 (BASELINE configs[0])"),
    "c2": dict(T=65536, B=8, D=1024, desc="C2 fp32 forward+backward linear recurrence T=65536 B=8 D=1024 (BASELINE configs[1])"),
    "c4": dict(T=1 << 20, B=1, D=128, desc="C4 fp32 1M-timestep recurrence T=1048576 B=1 D=128 (BASELINE configs[3])"),
    "c3": dict(T=65536, B=4, D=512, desc="C3 GILR-LSTM layer fwd+bwd T=65536 B=4 m=n=512 (BASELINE configs[2]): "
               "tensor-core gate GEMMs + fused scans"),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def traffic_from_profile(elements):
    """dram bytes per launch of the backward kernel from the committed
    `ncu --set full` summary (profiles/) when it was captured on this
    workload (same element count), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d["bwd"].get("elements_per_launch") != elements:
            return None
        return d["bwd"]["dram_bytes_per_launch"]
    except Exception:
        return None


OUR_KERNELS = re.compile(r"linrec_|\btc::|\blayers::|\btrain::")


def count_our_kernels(step, stream=None):
    """Kernels of this repository one call of step() launches, counted on the
    device with torch.profiler (CUPTI) in an untimed pass; None when the
    profiler is unavailable."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        return sum(1 for e in prof.events()
                   if e.device_type == torch.autograd.DeviceType.CUDA and OUR_KERNELS.search(e.name))
    except Exception:
        return None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1709_04057_b200 import capi

    world, rank, local = dist_env()
    # LINREC_BENCH_SHARE_GPU=1 (tests only): ranks share the visible GPUs and
    # talk over gloo, to exercise the N > 1 code paths on a 1-GPU box.
    share = os.environ.get("LINREC_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = WORKLOADS[args.workload]
    T, B, D = wl["T"], wl["B"], wl["D"]
    W = B * D
    seq_sharded = args.workload == "c4" and world > 1
    if seq_sharded:
        from paper_1709_04057_b200 import sharded
        Tl = sharded.segment_rows(T, world, rank)
    else:
        Tl = T
    N_local = Tl * W
    stream = torch.cuda.Stream(device=dev)
    st = stream.cuda_stream
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    with torch.cuda.stream(stream):
        lam = torch.empty(Tl, B, D, device=dev).uniform_(0.05, 0.95, generator=gen)
        x = torch.empty(Tl, B, D, device=dev).uniform_(-1.0, 1.0, generator=gen)
        h0 = torch.empty(B, D, device=dev).uniform_(-1.0, 1.0, generator=gen)
        dh = torch.empty(Tl, B, D, device=dev).uniform_(-1.0, 1.0, generator=gen)
        h = torch.empty_like(lam)
        dlam = torch.empty_like(lam)
        dx = torch.empty_like(lam)
        dh0 = torch.empty_like(h0)
    ws = capi.Workspace(local)
    stream.synchronize()

    if seq_sharded:
        runner = sharded.SequenceShardedScan(T, W, dist.group.WORLD, ws=ws, stream=stream)

        def fwd():
            runner.forward(lam, x, h0 if rank == 0 else None, h)

        def bwd():
            runner.backward(lam, h0 if rank == 0 else None, h, dh, dlam, dx, dh0)
        launches_per_step = runner.launches_per_step
    else:
        def fwd():
            capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), h.data_ptr(), Tl, W,
                      capi.PARALLEL, 4, ws.handle, st)

        def bwd():
            capi.scan_backward(lam.data_ptr(), h0.data_ptr(), h.data_ptr(), dh.data_ptr(),
                               dlam.data_ptr(), dx.data_ptr(), dh0.data_ptr(), Tl, W,
                               capi.PARALLEL, 4, ws.handle, st)
        launches_per_step = capi.scan_kernel_count(Tl, W, False) + capi.scan_kernel_count(Tl, W, True)

    # correctness guard (bench.hpp:204-216 analogue, untimed): chained scan vs
    # the bit-exact serial kernel on the same device inputs.
    if not seq_sharded:
        with torch.cuda.stream(stream):
            fwd()
            hs = torch.empty_like(h)
            capi.scan(lam.data_ptr(), x.data_ptr(), h0.data_ptr(), hs.data_ptr(), Tl, W,
                      capi.SERIAL, 4, None, st)
            err = ((h - hs).abs().max() / hs.abs().max().clamp_min(1.0)).item()
            del hs
        if err > 2e-4:
            raise SystemExit(f"bench guard: chained vs serial disagreement {err:.3e}")

    for _ in range(args.warmup):
        fwd()
        bwd()
    # kernels per step counted on the device (untimed); the planner's count as fallback
    counted = count_our_kernels(lambda: (fwd(), bwd()))
    if counted is not None:
        launches_per_step = counted
    n_ev = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_ev)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            fwd()
            ev[i][1].record(stream)
            bwd()
            ev[i][2].record(stream)
        end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(end)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in ev]
    if world > 1:
        t = torch.tensor([total_ms], device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    ms_step = total_ms / args.steps
    N_total = (T * W) if seq_sharded else N_local * world
    value = N_total / (ms_step / 1e3)

    peak, peak_kind = peaks()
    fwd_avg = statistics.mean(fwd_ms)
    bwd_avg = statistics.mean(bwd_ms)
    fwd_gbs = FWD_BYTES * N_local / (fwd_avg / 1e3) / 1e9
    bwd_gbs = BWD_BYTES * N_local / (bwd_avg / 1e3) / 1e9
    step_gbs = (FWD_BYTES + BWD_BYTES) * N_local / (ms_step / 1e3) / 1e9 if not seq_sharded else \
        (FWD_BYTES + BWD_BYTES) * N_local / (ms_step / 1e3) / 1e9
    traffic = traffic_from_profile(N_local)

    result = None
    if rank == 0:
        result = {
            "metric": METRIC,
            "value": value,
            "unit": "elements/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong" if seq_sharded else "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic: lam~U(0.05,0.95), x,h0,dh~U(-1,1) (bench.hpp:134-143), torch RNG on device",
            "config": {
                "workload": wl["desc"],
                "T": T, "B": B, "D": D, "elements_per_step": N_total,
                "parallelism": ("sequence-sharded x%d (carry exchange: %s)" % (
                    world, "peer-memory mailboxes over NVLink" if runner.exchange == "p2p" else "all-gather"))
                if seq_sharded
                else ("single GPU" if world == 1 else "channel-sharded x%d (independent [T,W] blocks, no collective)" % world),
                "l2": "no flush: every tensor is %.0f MiB >> 126 MB L2" % (N_local * 4 / 2**20),
                "timing": "CUDA events on the launching stream, max over ranks",
            },
            "hbm_gbs": step_gbs,
            "pct_of_peak": 100.0 * step_gbs / peak,
            "kernels": {
                "fwd": {"ms": fwd_avg, "gbs": fwd_gbs, "bytes_per_element": FWD_BYTES},
                "bwd": {"ms": bwd_avg, "gbs": bwd_gbs, "bytes_per_element": BWD_BYTES},
            },
            "roofline": {
                "bound": "hbm",
                "kernel": "k_tma_bwd (persistent TMA-fed reverse-time chained scan, fused dlam/dx/dh0)",
                "achieved": bwd_gbs,
                "peak": peak,
                "peak_kind": peak_kind,
                "unit": "GB/s",
                "frac": bwd_gbs / peak,
                "traffic": traffic,
                "algorithmic_bytes_per_launch": BWD_BYTES * N_local,
                "fwd": {"achieved": fwd_gbs, "frac": fwd_gbs / peak, "algorithmic_bytes_per_launch": FWD_BYTES * N_local},
            },
            "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_method": "kernels of this repo per step counted with torch.profiler (CUPTI) over one untimed step, x steps",
            "clocks": clocks.summary(),
        }
    # free device memory before the e2e leg
    del lam, x, h0, dh, h, dlam, dx, dh0
    torch.cuda.empty_cache()
    if world > 1:
        dist.barrier()
    e2e = None
    if not args.no_e2e and not seq_sharded:
        e2e = e2e_leg(args, T, B, D, local, world, share)
    if rank == 0:
        if e2e is not None:
            result["e2e"] = e2e
        if not args.no_cpu and world == 1:
            result["cpu_baseline"] = cpu_baseline_leg(args, T, B, D)
        print(json.dumps(result), flush=True)
    if world > 1:
        if seq_sharded:
            runner.close()
        dist.barrier()
        dist.destroy_process_group()


def e2e_leg(args, T, B, D, device, world=1, share=False):
    """Same metric through the host-pointer C ABI from pinned host memory; at
    N > 1 every rank runs its own block concurrently (max time over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1709_04057_b200 import capi

    W = B * D
    N = T * W
    shape = (T, B, D)
    pin = lambda s: torch.empty(s, dtype=torch.float32, pin_memory=True)  # noqa: E731
    lam, x, dh, h, dlam, dx = (pin(shape) for _ in range(6))
    h0, dh0 = pin((B, D)), pin((B, D))
    rng = np.random.default_rng(5)
    chunk = 1 << 14
    for t0 in range(0, T, chunk):  # fill without a 2 GiB temporary
        sl = slice(t0, min(T, t0 + chunk))
        n = (sl.stop - sl.start, B, D)
        lam[sl].numpy()[:] = rng.uniform(0.05, 0.95, n)
        x[sl].numpy()[:] = rng.uniform(-1, 1, n)
        dh[sl].numpy()[:] = rng.uniform(-1, 1, n)
    h0.numpy()[:] = rng.uniform(-1, 1, (B, D))
    p = lambda t: t.data_ptr()  # noqa: E731

    def step():
        capi.scan_host(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, device)
        capi.scan_backward_host(p(lam), p(h0), p(h), p(dh), p(dlam), p(dx), p(dh0), T, W,
                                capi.PARALLEL, 4, device)

    steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(max(1, min(args.warmup, 2))):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        t = torch.tensor([dt], device="cpu" if share else torch.device("cuda", device))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = t.item()
    return {
        "value": world * N / dt,
        "unit": "elements/s",
        "ms_per_step": dt * 1e3,
        "steps": steps,
        # per rank x ranks; fwd: lam, x, h0 in / h out; bwd: lam, h, dh, h0 in / dlam, dx, dh0 out
        "h2d_bytes_per_step": world * (4 * (2 * N + W) + 4 * (3 * N + W)),
        "d2h_bytes_per_step": world * (4 * N + 4 * (2 * N + W)),
        "api": "linrec_scan_host_f32 + linrec_scan_backward_host_f32 (the numpy boundary of linrec.scan / linrec.scan_backward), pinned buffers",
        "timing": "host wall clock, synchronous calls, max over ranks",
        "ranks": world,
    }


def cpu_baseline_leg(args, T, B, D):
    """The reference's CPU implementation (oracle/_ref) on this host's cores,
    bounded sample, bench.hpp:93-107 protocol."""
    import numpy as np
    try:
        from oracle.oracle import RefLib
        ref = RefLib()
    except Exception as e:
        return {"value": None, "unit": "elements/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}
    cores = os.cpu_count() or 1
    Ts = min(T, args.cpu_rows)
    rng = np.random.default_rng(7)
    lam = rng.uniform(0.05, 0.95, (Ts, B, D)).astype(np.float32)
    x = rng.uniform(-1, 1, (Ts, B, D)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (B, D)).astype(np.float32)
    dh = rng.uniform(-1, 1, (Ts, B, D)).astype(np.float32)
    f, b = ref.bench_fwd_bwd(lam, x, h0, dh, cores, warmup=1, reps=args.cpu_reps)
    n = Ts * B * D
    return {
        "value": n / (f + b),
        "unit": "elements/s",
        "cores": cores,
        "kind": "reference",
        "sample": (f"T={Ts} of {T} rows x B={B} x D={D} ({n} elements): reference scan_parallel + "
                   f"scan_backward(ScanMode::Parallel), workers={cores}, median of {args.cpu_reps} reps"),
        "fwd_elements_per_s": n / f,
        "bwd_elements_per_s": n / b,
    }


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation through its public
# Python API (oracle/_ref/linrec*.so = proj/bindings/linrec_py.cpp compiled
# from /root/reference), on this host's cores.
# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    wl = WORKLOADS[args.workload]
    T, B, D = wl["T"], wl["B"], wl["D"]
    try:
        from oracle.oracle import load_reference_module
        ref = load_reference_module()
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    cores = os.cpu_count() or 1
    Ts = min(T, args.cpu_rows)
    rng = np.random.default_rng(7)
    lam = rng.uniform(0.05, 0.95, (Ts, B, D)).astype(np.float32)
    x = rng.uniform(-1, 1, (Ts, B, D)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (B, D)).astype(np.float32)
    dh = rng.uniform(-1, 1, (Ts, B, D)).astype(np.float32)

    def step():
        h = ref.scan(lam, x, h0, workers=cores)
        ref.scan_backward(lam, h0, h, dh, workers=cores)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    n = Ts * B * D
    value = n / (ms / 1e3)
    sample = (f"T={Ts} of {T} rows x B={B} x D={D} ({n} elements) per step: linrec.scan + "
              f"linrec.scan_backward (reference pybind11 API, numpy in/out), workers={cores}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: lam~U(0.05,0.95), x,h0,dh~U(-1,1)",
        "config": {"workload": wl["desc"], "T": T, "B": B, "D": D, "sampled_rows": Ts},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# C3: one GILR-LSTM layer forward + backward (layers.hpp:245-375)
# ---------------------------------------------------------------------------
def layer_stage_work(T, b, m, n):
    """Algorithmic work per stage: ("flop", 2*M*N*K) for the GEMMs, ("byte",
    bytes) for the scans and pointwise passes (fp32)."""
    R = T * b
    E = R * n
    return {
        "gemm_surrogate": ("flop", 2 * R * m * 2 * n),
        "scan_surrogate": ("byte", 12 * E),
        "gemm_gates": ("flop", 2 * R * (m + n) * 4 * n),
        "scan_cell": ("byte", 12 * E),
        "h_out": ("byte", 12 * E),
        "dc": ("byte", 12 * E),
        "scan_bwd_cell": ("byte", 16 * E),       # dlam not stored: dpre forms it from c
        "dpre_gates": ("byte", 44 * E),          # f i o z diz dh c in, 4 dpre planes out
        "wgrad_U": ("flop", 2 * 4 * n * n * R),
        "wgrad_V": ("flop", 2 * 4 * n * m * R),
        "dhtil_prev": ("flop", 2 * R * 4 * n * n),
        "scan_bwd_surrogate": ("byte", 16 * E),
        "dpre_surrogate": ("byte", 24 * E),
        "wgrad_surrogate_U": ("flop", 2 * n * m * R),
        "wgrad_surrogate_V": ("flop", 2 * n * m * R),
        "dx": ("flop", 2 * R * m * 6 * n),
    }


def tensor_peak():
    """Dense TF32 tensor-core peak for the roofline: the nominal 1.1 PFLOP/s
    of B200_PROFILING.md.  MEASURED_PEAKS.json has no TF32 figure, and half of
    its measured bf16 rate (cuBLAS) is no upper bound here: the 3xTF32 GEMMs
    issue MMAs at ~900 TF/s with the split disabled."""
    return 1100.0, "nominal dense TF32 (B200_PROFILING.md); no measured TF32 peak exists"


def run_layer(args):
    import torch
    from paper_1709_04057_b200 import layers as L

    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("c3 is a single-GPU workload (the layer shards like C2 over channels: run replicas)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    wl = WORKLOADS["c3"]
    T, b, n = wl["T"], wl["B"], wl["D"]
    m = n
    prec = args.precision
    stream = torch.cuda.Stream(device=dev)
    gen = torch.Generator().manual_seed(7)
    with torch.cuda.stream(stream):
        p = L.gilr_lstm_init(gen, m, n, 1.0, dev)
        g = torch.Generator(device=dev).manual_seed(11)
        x = torch.empty(T, b, m, device=dev).uniform_(-1, 1, generator=g)
        dh = torch.empty(T, b, n, device=dev).uniform_(-1, 1, generator=g)
        z = torch.zeros(b, n, device=dev)
        cache = L.GilrLstmCache()
        grads = L.GilrLstmGrads.zeros_like(p)

        def step():
            for t in grads.tensors():
                t.zero_()
            h = L.gilr_lstm_forward(p, x, z, z, precision=prec, cache=cache)
            dx, _, _ = L.gilr_lstm_backward(p, x, z, z, cache, dh, grads, precision=prec)
            return h, dx

        for _ in range(args.warmup):
            step()
        # correctness guard (untimed; bench.hpp:375-384 analogue): the same
        # layer forward with the per-channel serial scans vs the chained ones
        h_par = L.gilr_lstm_forward(p, x, z, z, precision=prec, cache=L.GilrLstmCache())
        h_ser = L.gilr_lstm_forward(p, x, z, z, mode="serial", precision=prec, cache=L.GilrLstmCache())
        guard = ((h_par - h_ser).abs().max() / h_ser.abs().max().clamp_min(1.0)).item()
        del h_par, h_ser
        if guard > 2e-4:
            raise SystemExit(f"bench guard: serial/parallel layer disagreement {guard:.3e}")
    stream.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L.profile_begin()
    with ClockSampler(local) as clocks, torch.cuda.stream(stream):
        start.record(stream)
        for _ in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize(dev)
    stages = L.profile_end()
    ms = start.elapsed_time(end) / args.steps
    E = T * b * n
    work = layer_stage_work(T, b, m, n)
    hbm, hbm_kind = peaks()
    tpk, tpk_kind = tensor_peak()
    st_out, best = {}, None
    for name, (tot, cnt) in stages.items():
        avg = tot / args.steps
        rec = {"ms": avg, "launch_sets_per_step": cnt / args.steps}
        if name in work:
            kind, amount = work[name]
            if kind == "flop":
                rec["tflops"] = amount / (avg / 1e3) / 1e12
                rec["frac_tf32_peak"] = rec["tflops"] / tpk
                rec["mma_issue_frac"] = rec["frac_tf32_peak"] * (3 if prec == "fp32" else 1)
                if best is None or avg > best[1]:
                    best = (name, avg, amount)
            else:
                rec["gbs"] = amount / (avg / 1e3) / 1e9
                rec["frac_hbm_peak"] = rec["gbs"] / hbm
        st_out[name] = rec
    gemm_ms = sum(v["ms"] for k, v in st_out.items() if "tflops" in v)
    flops = sum(a for k, (kind, a) in work.items() if kind == "flop")
    bname, bms, bflop = best
    achieved = bflop / (bms / 1e3) / 1e12
    result = {
        "metric": METRIC,
        "value": E / (ms / 1e3),
        "unit": "elements/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (GEMMs: %s)" % ("3xTF32 tcgen05, fp32-grade" if prec == "fp32" else "TF32 tcgen05"),
        "data": "synthetic: x, d_h ~U(-1,1); parameters from gilr_lstm_init (layers.hpp:165-176), gate_bias 1",
        "config": {
            "workload": wl["desc"], "T": T, "B": b, "m": m, "n": n, "elements_per_step": E,
            "events_per_step": T * b, "precision": prec,
            "step": "zero grads + gilr_lstm_forward + gilr_lstm_backward (one layer)",
            "guard_serial_vs_parallel": guard,
            "l2": "no flush: activations are %.0f MiB per [T,b,n] tensor >> 126 MB L2" % (E * 4 / 2**20),
            "timing": "CUDA events on the launching stream; per-stage events via linrec_profile_begin/end",
        },
        "events_per_s": T * b / (ms / 1e3),
        "gemm_tflops_total": flops / (gemm_ms / 1e3) / 1e12,
        "gemm_share_of_step": gemm_ms / ms,
        "stages": st_out,
        "roofline": {
            "bound": "tensor",
            "kernel": f"k_gemm ({bname}) -- the longest tensor-core stage",
            "achieved": achieved,
            "peak": tpk,
            "peak_kind": tpk_kind,
            "unit": "TFLOP/s",
            "frac": achieved / tpk,
            # 3xTF32 issues three MMAs per algorithmic product
            "mma_issue_frac": (3 if prec == "fp32" else 1) * achieved / tpk,
            "effective_peak_for_precision": tpk / (3 if prec == "fp32" else 1),
            "traffic": None,
            "algorithmic_flops_per_launch": bflop,
        },
        "gpu_launches": None,
        "clocks": clocks.summary(),
    }
    # kernels per step counted on the device with torch.profiler (untimed pass)
    counted = count_our_kernels(step)
    result["gpu_launches"] = (counted * args.steps if counted is not None
                              else sum(round(v["launch_sets_per_step"]) for v in st_out.values()) * args.steps)
    result["gpu_launches_method"] = ("kernels of this repo per step counted with torch.profiler (CUPTI) over one "
                                     "untimed step, x steps" if counted is not None else "stage call count")
    del cache, grads
    torch.cuda.empty_cache()
    if not args.no_e2e:
        result["e2e"] = layer_e2e(args, p, T, b, m, n, dev)
    if not args.no_cpu:
        result["cpu_baseline"] = layer_cpu_baseline(args, m, n, b)
    print(json.dumps(result), flush=True)


def layer_e2e(args, p, T, b, m, n, dev):
    """Host x, d_h (pinned) -> device -> forward + backward -> h, dx back to host."""
    import torch
    from paper_1709_04057_b200 import layers as L
    xh = torch.empty(T, b, m, pin_memory=True).uniform_(-1, 1)
    dhh = torch.empty(T, b, n, pin_memory=True).uniform_(-1, 1)
    hh = torch.empty(T, b, n, pin_memory=True)
    dxh = torch.empty(T, b, m, pin_memory=True)
    z = torch.zeros(b, n, device=dev)
    cache = L.GilrLstmCache()
    grads = L.GilrLstmGrads.zeros_like(p)

    def step():
        x = xh.to(dev, non_blocking=True)
        dh = dhh.to(dev, non_blocking=True)
        for t in grads.tensors():
            t.zero_()
        h = L.gilr_lstm_forward(p, x, z, z, precision=args.precision, cache=cache)
        dx, _, _ = L.gilr_lstm_backward(p, x, z, z, cache, dh, grads, precision=args.precision)
        hh.copy_(h, non_blocking=True)
        dxh.copy_(dx, non_blocking=True)
        torch.cuda.synchronize(dev)

    step()
    steps = max(1, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    return {"value": T * b * n / dt, "unit": "elements/s", "ms_per_step": dt * 1e3, "steps": steps,
            "h2d_bytes_per_step": 4 * T * b * (m + n), "d2h_bytes_per_step": 4 * T * b * (n + m),
            "api": "paper_1709_04057_b200.layers.gilr_lstm_forward/backward (C ABI linrec_gilr_lstm_*_f32)",
            "timing": "host wall clock incl. pinned H2D of x, d_h and D2H of h, dx"}


def layer_cpu_baseline(args, m, n, b):
    """The oracle port of layers.hpp (oracle/linrec_layers.c, fp32, 1 thread)
    on a bounded sample: the reference's own layer path needs Eigen, which is
    absent here."""
    import numpy as np
    from oracle.oracle import Oracle, gilr_lstm_params
    orc = Oracle()
    Ts = args.layer_cpu_rows
    rng = np.random.default_rng(3)
    P = {k: v.astype(np.float32) for k, v in gilr_lstm_params(rng, m, n).items()}
    x = rng.uniform(-1, 1, (Ts, b, m)).astype(np.float32)
    dh = rng.uniform(-1, 1, (Ts, b, n)).astype(np.float32)
    z = np.zeros((b, n), np.float32)
    t0 = time.perf_counter()
    h, cache = orc.gilr_lstm_forward(P, x, z, z)
    orc.gilr_lstm_backward(P, x, z, z, cache, dh)
    dt = time.perf_counter() - t0
    return {"value": Ts * b * n / dt, "unit": "elements/s", "cores": 1, "kind": "port",
            "sample": f"T={Ts} rows x b={b} x m=n={n}: oracle gilr_lstm_forward + gilr_lstm_backward "
                      f"(plain-C restatement of layers.hpp, naive loops), fp32, 1 thread, {dt:.1f} s"}


def run_reference_layer(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    wl = WORKLOADS["c3"]
    T, b, n = wl["T"], wl["B"], wl["D"]
    for _ in range(max(0, min(args.warmup, 1))):
        pass
    reps = [layer_cpu_baseline(args, n, n, b) for _ in range(max(1, min(args.steps, 2)))]
    v = statistics.median(r["value"] for r in reps)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s", "n_gpus": world,
        "steps": len(reps), "warmup": 0, "ms_per_step": 1e3 * args.layer_cpu_rows * b * n / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": wl["desc"], "T": T, "B": b, "m": n, "n": n,
                                        "sampled_rows": args.layer_cpu_rows},
        "cpu_baseline": dict(reps[0], value=v),
        "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference's layer path needs Eigen (absent; SURVEY.md 8c): its oracle port is timed",
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=4096)
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precision", choices=["fp32", "tf32"], default="fp32", help="c3 GEMM precision")
    ap.add_argument("--layer-cpu-rows", type=int, default=16)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.workload == "c3":
        run_reference_layer(args) if args.impl == "reference" else run_layer(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
