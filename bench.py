#!/usr/bin/env python
"""Benchmark of the linear-recurrence hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c4|c1|c3|c5] [--precision fp32|tf32]

One step = one forward scan (lam, x, h0 -> h) + one reverse-time backward scan
(lam, h0, h, dh -> dlam, dx, dh0) over one batch of synthetic input, fp32.
Default workload = BASELINE configs[1] ("C2"): T=65536, B=8, D=1024.

* ``value``      elements/s fwd+bwd (N_elements / step time), inputs resident in
                 HBM, device-timed with CUDA events on the launching stream
                 around exactly K steps, max over ranks; each tensor is 2 GiB
                 >> the 126 MB L2, so no flush is needed between steps.  An
                 untimed guard re-runs a channel subset over the full sequence
                 with the bit-exact serial kernels (<= 1e-5 or the run fails).
* ``slow_decay`` the same with lam ~ U(0.99, 1) (the fix-up's worst case).
* ``c4`` / ``c4_seq_sharded``  the 1M-step workload (configs[3]) beside the
                 headline: 1 GPU, and at N > 1 sequence-sharded over all ranks
                 with its strong-scaling speed-up over rank 0 alone.
* ``e2e``        the same metric through the reference's Python API
                 (``linrec.scan`` / ``linrec.scan_backward``) on pageable numpy
                 arrays, outputs allocated per call; ``e2e.pinned`` the C ABI
                 host entry points from pinned buffers.
* ``roofline``   dominant kernel (the backward scan: 20 of the 32 algorithmic
                 B/element) -- algorithmic bytes / measured launch time vs the
                 measured HBM copy peak (MEASURED_PEAKS.json).
* ``cpu_baseline`` the reference's own CPU path (oracle/_ref, compiled from
                 /root/reference) on this host's cores, on the GPU arm's exact
                 inputs, whole problem; plus its 1-core serial path.

--gpus N without torchrun re-executes itself under torch.distributed.run (one
rank per GPU).  Multi-GPU: c2 is channel-sharded (each rank an independent
[T, W] block, no data-path collective; weak scaling); c4 is sequence-sharded
with a peer-memory carry exchange (strong scaling); c5 (2^28 elements per
(T, W) point) shards channels at large W and the sequence at small W.
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
# the roofline line's dominant kernel (the backward), by the family the library
# picks for the shape (capi.scan_kernel_name)
BWD_KERNEL_DESC = {
    "tma": "k_tma_bwd (persistent TMA-fed reverse-time chained scan, fused dlam/dx/dh0)",
    "chained": "k_chain_bwd (register-tiled reverse-time chained scan, fused dlam/dx/dh0)",
    "cluster": "k_cluster_bwd (thread-block cluster over the sequence, DSMEM carry exchange, fused dlam/dx/dh0)",
    "local": "k_local_bwd (CTA-local reverse-time scan, fused dlam/dx/dh0)",
    "serial": "k_serial_bwd (per-channel reverse-time scan)",
}
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
# synthetic inputs (bench.hpp:134-143 distributions), generated on the host
# so the GPU arm, the e2e leg, the CPU baseline and the reference arm see the
# SAME numbers; a global [T, ...] array is defined independently of how many
# ranks share it (fixed row blocks, one PCG64 stream per block).
# ---------------------------------------------------------------------------
LAM_BENCH = (0.05, 0.95)   # bench.hpp:134-143
LAM_SLOW = (0.99, 1.0)     # slow decays: the fix-up walks whole segments


def host_rows(T, row_shape, lo, hi, seed, r0=0, r1=None):
    """Rows [r0, r1) of a global float32 [T, *row_shape] array ~ U(lo, hi)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    r1 = T if r1 is None else r1
    W = 1
    for d in row_shape:
        W *= d
    bs = max(1, -(-T // 256))
    nb = -(-T // bs)
    seqs = np.random.SeedSequence(seed).spawn(nb)
    out = np.empty((r1 - r0,) + tuple(row_shape), np.float32)
    flat = out.reshape(r1 - r0, W)

    def fill(k):
        s, e = k * bs, min(T, (k + 1) * bs)
        a, b = max(s, r0), min(e, r1)
        if a >= b:
            return
        g = np.random.Generator(np.random.PCG64(seqs[k]))
        dst = flat[a - r0:b - r0]
        if (a, b) == (s, e):
            g.random(out=dst, dtype=np.float32)
        else:
            dst[:] = g.random((e - s, W), dtype=np.float32)[a - s:b - s]
        dst *= np.float32(hi - lo)
        dst += np.float32(lo)

    with ThreadPoolExecutor(max(1, min(16, os.cpu_count() or 1))) as ex:
        list(ex.map(fill, range(nb)))
    return out


def host_problem(T, B, D, seed, r0=0, r1=None, lam=LAM_BENCH):
    """(lam, x, h0, dh) rows [r0, r1) of the global problem `seed`; h0 is the
    global [B, D] initial state."""
    return (host_rows(T, (B, D), lam[0], lam[1], seed * 10 + 1, r0, r1),
            host_rows(T, (B, D), -1.0, 1.0, seed * 10 + 2, r0, r1),
            host_rows(1, (B, D), -1.0, 1.0, seed * 10 + 3)[0],
            host_rows(T, (B, D), -1.0, 1.0, seed * 10 + 4, r0, r1))


SEED_C2, SEED_C4 = 1000, 4000


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# process group plumbing
# ---------------------------------------------------------------------------
class Ranks:
    """world / rank / device; gloo when ranks share one GPU (tests)."""

    def __init__(self):
        import torch
        import torch.distributed as dist
        self.world, self.rank, self.local = dist_env()
        # LINREC_BENCH_SHARE_GPU=1 (tests only): ranks share the visible GPUs and
        # talk over gloo, to exercise the N > 1 code paths on a 1-GPU box.
        self.share = os.environ.get("LINREC_BENCH_SHARE_GPU") == "1"
        if self.share:
            self.local = self.local % max(1, torch.cuda.device_count())
        if self.world > 1:
            if self.share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()

    def max(self, v):
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device="cpu" if self.share else self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def gather(self, obj):
        import torch.distributed as dist
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def bcast(self, obj):
        import torch.distributed as dist
        if self.world == 1:
            return obj
        lst = [obj]
        dist.broadcast_object_list(lst, src=0)
        return lst[0]

    def close(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
            dist.destroy_process_group()


class _FastLaunch:
    """The timed loop of a graph-replayed step through the driver API
    (cuGraphLaunch / cuEventRecord on the raw handles of the captured graph and
    the per-step events): each step is still one launch of the whole-step
    graph on the bench stream, bracketed by its two events, but the host no
    longer needs ~20 us of Python per step -- at C1 (14 us of device time per
    step) the GPU would otherwise wait on the host.  None when the handles
    are unavailable (the caller falls back to CUDAGraph.replay)."""

    def __init__(self, cu, exec_h, stream_h, events):
        self.cu, self.exec_h, self.stream_h, self.events = cu, exec_h, stream_h, events

    @staticmethod
    def make(step, stream, ev):
        import ctypes as C
        try:
            exec_h = step.graph.raw_cuda_graph_exec()
            if not isinstance(exec_h, int) or exec_h == 0:
                return None
            cu = C.CDLL("libcuda.so.1")
            cu.cuGraphLaunch.argtypes = [C.c_void_p, C.c_void_p]
            cu.cuEventRecord.argtypes = [C.c_void_p, C.c_void_p]
            for e in ev:  # torch creates the CUDA events at their first record
                e[0].record(stream)
                e[2].record(stream)
            events = [(e[0].cuda_event, e[2].cuda_event) for e in ev]
            if any(a == 0 or b == 0 for a, b in events):
                return None
            return _FastLaunch(cu, exec_h, stream.cuda_stream, events)
        except Exception:  # noqa: BLE001 -- older torch: keep replay()
            return None

    def run(self, steps):
        rec, launch, g, st = self.cu.cuEventRecord, self.cu.cuGraphLaunch, self.exec_h, self.stream_h
        for i in range(steps):
            a, b = self.events[i]
            if rec(a, st) or launch(g, st) or rec(b, st):
                raise RuntimeError("bench: cuGraphLaunch / cuEventRecord failed")


def time_steps(rk, fwd, bwd, steps, stream, step=None):
    """EXACTLY `steps` steps between a barrier + synchronize on both sides,
    CUDA events on the launching stream, max over ranks; NVML clocks sampled
    during the timed region.  With `step` (single GPU: the whole fwd + bwd
    step as ONE CUDA graph) each timed step is one replay, and the fwd / bwd
    split comes from a short separate pass over the per-direction graphs
    (outside the timed region); otherwise (eager, sequence-sharded) the split
    is recorded inside the timed steps."""
    import torch
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    fast = _FastLaunch.make(step, stream, ev) if step is not None else None
    rk.barrier()
    torch.cuda.synchronize(rk.dev)
    with ClockSampler(rk.local) as clocks:
        start.record(stream)
        if fast is not None:
            fast.run(steps)  # the same replays, launched without Python-side overhead per step
        else:
            for i in range(steps):
                ev[i][0].record(stream)
                if step is not None:
                    step()
                else:
                    fwd()
                    ev[i][1].record(stream)
                    bwd()
                ev[i][2].record(stream)
        end.record(stream)
        torch.cuda.synchronize(rk.dev)
    rk.barrier()
    total = rk.max(start.elapsed_time(end))
    step_ms = [e[0].elapsed_time(e[2]) for e in ev]
    if step is not None:  # the split, from per-direction replays
        sp = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(min(steps, 10))]
        for e in sp:
            e[0].record(stream)
            fwd()
            e[1].record(stream)
            bwd()
            e[2].record(stream)
        torch.cuda.synchronize(rk.dev)
        split = sp
    else:
        split = ev
    fwd_ms = [e[0].elapsed_time(e[1]) for e in split]
    bwd_ms = [e[1].elapsed_time(e[2]) for e in split]
    return {
        "ms_per_step": total / steps,
        "median_ms_per_step": rk.max(statistics.median(step_ms)),
        "fwd_ms": rk.max(statistics.mean(fwd_ms)),
        "bwd_ms": rk.max(statistics.mean(bwd_ms)),
        "clocks": clocks.summary(),
    }


def rel_err(a, b):
    """max|a - b| / max|b| (oracles.hpp:73-82), on the device."""
    den = b.abs().max().item()
    num = (a.double() - b.double()).abs().max().item()
    return num / den if den else (0.0 if num == 0 else float("inf"))


# ---------------------------------------------------------------------------
# scan problems on the device: single GPU or sequence-sharded
# ---------------------------------------------------------------------------
class DeviceProblem:
    """lam, x, h0, dh (inputs) and h, dlam, dx, dh0 (outputs) on the device,
    [Tl, B, D] rows of a [T, B, D] problem."""

    def __init__(self, host, dev, stream):
        import torch
        lam, x, h0, dh = host
        with torch.cuda.stream(stream):
            self.lam, self.x, self.h0, self.dh = (torch.from_numpy(a).to(dev, non_blocking=False)
                                                  for a in (lam, x, h0, dh))
            self.h = torch.empty_like(self.lam)
            self.dlam = torch.empty_like(self.lam)
            self.dx = torch.empty_like(self.lam)
            self.dh0 = torch.empty_like(self.h0)
        stream.synchronize()
        self.Tl = self.lam.shape[0]
        self.W = self.lam[0].numel()

    def regen_lam(self, lo, hi, seed, stream):
        """Decays replaced in place (device RNG; the slow-decay variant), on the
        bench stream and finished before anything reads them."""
        import torch
        g = torch.Generator(device=self.lam.device).manual_seed(seed)
        with torch.cuda.stream(stream):
            self.lam.uniform_(lo, hi, generator=g)
        stream.synchronize()

    def free(self):
        for k in ("lam", "x", "h0", "dh", "h", "dlam", "dx", "dh0"):
            setattr(self, k, None)


def single_gpu_steps(P, ws, stream):
    """fwd / bwd of one step, each captured once into a CUDA graph and replayed
    (no host launch gaps between steps: the small workloads -- C1 is ~20 us
    per direction -- would otherwise time Python + ctypes overhead).  The
    workspace's control block is device-resident, so replays are exact
    re-launches (tests/test_gpu_parity.py::test_workspace_reuse_and_cuda_graph_replay).
    The eager callables are kept as .eager for the kernel count."""
    import torch
    from paper_1709_04057_b200 import capi
    st = stream.cuda_stream

    def fwd():
        capi.scan(P.lam.data_ptr(), P.x.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.Tl, P.W,
                  capi.PARALLEL, 4, ws.handle, st)

    def bwd():
        capi.scan_backward(P.lam.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.dh.data_ptr(),
                           P.dlam.data_ptr(), P.dx.data_ptr(), P.dh0.data_ptr(), P.Tl, P.W,
                           capi.PARALLEL, 4, ws.handle, st)
    fwd(), bwd()  # workspace sized before capture
    stream.synchronize()
    gf, gb, gs = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf, stream=stream):
        fwd()
    with torch.cuda.graph(gb, stream=stream):
        bwd()
    with torch.cuda.graph(gs, stream=stream):  # the whole step: one replay per step
        fwd()
        bwd()
    return _Replay(gf, fwd, stream), _Replay(gb, bwd, stream), _Replay(gs, None, stream)


def device_dir_ms(P, ws, stream, k=16, reps=5):
    """Per-launch device time of the forward and of the backward scan alone:
    k back-to-back launches of one direction in one graph, / k (median of
    reps) -- the roofline's kernel duration for short steps, where a
    one-launch replay's graph overhead (~4 us) would be charged to the
    kernel."""
    import torch
    from paper_1709_04057_b200 import capi
    st = stream.cuda_stream

    def f():
        capi.scan(P.lam.data_ptr(), P.x.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.Tl, P.W,
                  capi.PARALLEL, 4, ws.handle, st)

    def b():
        capi.scan_backward(P.lam.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.dh.data_ptr(),
                           P.dlam.data_ptr(), P.dx.data_ptr(), P.dh0.data_ptr(), P.Tl, P.W,
                           capi.PARALLEL, 4, ws.handle, st)
    out = []
    for fn in (f, b):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(k):
                fn()
        times = []
        with torch.cuda.stream(stream):
            g.replay()
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1) / k)
        out.append(statistics.median(times))
    return out


def device_ms_per_step(P, ws, stream, k=16, reps=5):
    import torch
    from paper_1709_04057_b200 import capi
    st = stream.cuda_stream
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(k):
            capi.scan(P.lam.data_ptr(), P.x.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.Tl, P.W,
                      capi.PARALLEL, 4, ws.handle, st)
            capi.scan_backward(P.lam.data_ptr(), P.h0.data_ptr(), P.h.data_ptr(), P.dh.data_ptr(),
                               P.dlam.data_ptr(), P.dx.data_ptr(), P.dh0.data_ptr(), P.Tl, P.W,
                               capi.PARALLEL, 4, ws.handle, st)
    times = []
    with torch.cuda.stream(stream):
        g.replay()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b) / k)
    return statistics.median(times)


class _Replay:
    """A captured graph replayed on the bench stream (CUDAGraph.replay
    launches on the CURRENT stream)."""

    def __init__(self, graph, eager, stream):
        self.graph, self.eager, self.stream = graph, eager, stream

    def __call__(self):
        import torch
        with torch.cuda.stream(self.stream):
            self.graph.replay()


def sharded_steps(rk, P, T, ws, stream):
    from paper_1709_04057_b200 import sharded
    import torch.distributed as dist
    runner = sharded.SequenceShardedScan(T, P.W, dist.group.WORLD, ws=ws, stream=stream)
    r = rk.rank

    def fwd():
        runner.forward(P.lam, P.x, P.h0 if r == 0 else None, P.h)

    def bwd():
        runner.backward(P.lam, P.h0 if r == 0 else None, P.h, P.dh, P.dlam, P.dx, P.dh0)
    return fwd, bwd, runner


def guard(rk, P, stream, cols=8):
    """Untimed correctness guard (the bench.hpp:204-216 analogue): a channel
    subset over the FULL sequence -- every rank's rows gathered on rank 0 --
    re-run with the bit-exact per-channel serial kernels (pinned to the
    reference by the parity tests) and compared with what the timed path
    produced.  Returns the max normwise error over h, dlam, dx, dh0."""
    import numpy as np
    import torch
    from paper_1709_04057_b200 import capi
    W = P.W
    with torch.cuda.stream(stream):  # idx on the same stream as its users (no cross-stream read)
        idx = torch.arange(0, W, max(1, W // cols), device=P.lam.device)[:cols]
        part = [t.view(t.shape[0], W).index_select(1, idx).cpu().numpy()
                for t in (P.lam, P.x, P.dh, P.h, P.dlam, P.dx)]
        h0s = P.h0.view(W).index_select(0, idx).cpu().numpy()
        dh0s = P.dh0.view(W).index_select(0, idx).cpu().numpy()
    parts = rk.gather(part)
    err = None
    if rk.rank == 0:
        full = [np.ascontiguousarray(np.concatenate([p[i] for p in parts])) for i in range(6)]
        L, X, DH, H, DL, DX = (torch.from_numpy(a).to(rk.dev) for a in full)
        H0, DH0 = torch.from_numpy(h0s).to(rk.dev), torch.from_numpy(dh0s).to(rk.dev)
        T, n = L.shape
        st = torch.cuda.current_stream(rk.dev).cuda_stream
        hs, dls, dxs, dh0r = (torch.empty_like(L), torch.empty_like(L), torch.empty_like(L),
                              torch.empty_like(H0))
        capi.scan(L.data_ptr(), X.data_ptr(), H0.data_ptr(), hs.data_ptr(), T, n, capi.SERIAL, 4, None, st)
        capi.scan_backward(L.data_ptr(), H0.data_ptr(), hs.data_ptr(), DH.data_ptr(), dls.data_ptr(),
                           dxs.data_ptr(), dh0r.data_ptr(), T, n, capi.SERIAL, 4, None, st)
        torch.cuda.synchronize(rk.dev)
        errs = {"h": rel_err(H, hs), "dlam": rel_err(DL, dls), "dx": rel_err(DX, dxs), "dh0": rel_err(DH0, dh0r)}
        err = max(errs.values())
        if not err <= GUARD_TOL:  # diagnostics: where the timed path's results differ
            for nm, a, b in (("h", H, hs), ("dlam", DL, dls), ("dx", DX, dxs)):
                bad = ((a - b).abs() > GUARD_TOL * max(1.0, b.abs().max().item())).nonzero()
                if len(bad):
                    print(f"bench guard: {nm} differs at {len(bad)} of {a.numel()} sampled elements; rows "
                          f"{bad[:, 0].min().item()}..{bad[:, 0].max().item()}, sampled channels "
                          f"{sorted(set(idx[bad[:, 1]].tolist()))[:8]} (T={T}, W={W}, errors {errs})",
                          file=sys.stderr, flush=True)
    return rk.bcast(err)


GUARD_TOL = 1e-5  # the north star's fp32 tolerance (test_smoke.py:35)


def check_guard(err, what):
    if err is None or not (err <= GUARD_TOL):
        raise SystemExit(f"bench guard ({what}): max normwise error {err} > {GUARD_TOL}")


def run_problem(rk, P, T, args, stream, ws, sharded_run, steps=None, count=False):
    """Warm-up, guard and the timed region for one problem; returns the
    timing record (+ the runner for sharded runs)."""
    st = stream.cuda_stream
    runner = None
    step = None
    if sharded_run:
        fwd, bwd, runner = sharded_steps(rk, P, T, ws, stream)
    else:
        fwd, bwd, step = single_gpu_steps(P, ws, stream)
    for _ in range(args.warmup):
        fwd()
        bwd()
    # sequence-sharded: rank 0 checks the gathered full sequence; otherwise
    # every rank checks its own independent block
    g = guard(rk, P, stream) if sharded_run else rk.max(guard(_Solo(rk), P, stream))
    rec = time_steps(rk, fwd, bwd, steps or args.steps, stream, step=step)
    rec["guard_max_rel_err"] = g
    if step is not None and rec["ms_per_step"] < 0.2:
        # a step this short is bound by the host's graph replay (~10 us from
        # Python): also report the device time per step with 16 steps in one
        # graph (informational; `ms_per_step` stays one replay per step)
        rec["device_ms_per_step"] = device_ms_per_step(P, ws, stream)
        rec["fwd_kernel_ms"], rec["bwd_kernel_ms"] = device_dir_ms(P, ws, stream)
    if count:
        n = count_our_kernels(lambda: (getattr(fwd, "eager", fwd)(), getattr(bwd, "eager", bwd)()))
        rec["launches_per_step"] = n
    if runner is not None:
        rec["exchange"] = runner.exchange
        runner.close()
    return rec


def summarize(rec, N_total, N_local, peak):
    ms = rec["ms_per_step"]
    out = {
        "value": N_total / (ms / 1e3),
        "ms_per_step": ms,
        "median_ms_per_step": rec["median_ms_per_step"],
        "fwd_ms": rec["fwd_ms"],
        "bwd_ms": rec["bwd_ms"],
        "hbm_gbs_per_gpu": (FWD_BYTES + BWD_BYTES) * N_local / (ms / 1e3) / 1e9,
        "guard_max_rel_err": rec["guard_max_rel_err"],
    }
    out["frac_of_peak_per_gpu"] = out["hbm_gbs_per_gpu"] / peak
    if "device_ms_per_step" in rec:  # short steps: the device time with 16 steps per graph
        d = rec["device_ms_per_step"]
        out["device_ms_per_step"] = d
        out["device_value"] = N_total / (d / 1e3)
        out["device_frac_of_peak_per_gpu"] = (FWD_BYTES + BWD_BYTES) * N_local / (d / 1e3) / 1e9 / peak
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    from paper_1709_04057_b200 import capi

    rk = Ranks()
    world, rank = rk.world, rk.rank
    wl = WORKLOADS[args.workload]
    T, B, D = wl["T"], wl["B"], wl["D"]
    W = B * D
    seq_sharded = args.workload == "c4" and world > 1
    stream = torch.cuda.Stream(device=rk.dev)
    st = stream.cuda_stream
    ws = capi.Workspace(rk.local)
    peak, peak_kind = peaks()

    # the headline problem: c2 -> every rank its own [T, B, D] block (channel
    # sharding: no collective, weak scaling); c4 -> rank r rows of the global
    # problem (sequence sharding, strong scaling)
    if seq_sharded:
        from paper_1709_04057_b200 import sharded
        r0, r1 = sharded.segment_bounds(T, world, rank)
        host = host_problem(T, B, D, SEED_C4, r0, r1)
    else:
        seed = (SEED_C4 if args.workload == "c4" else SEED_C2) + (rank if world > 1 else 0)
        host = host_problem(T, B, D, seed)
    P = DeviceProblem(host, rk.dev, stream)
    N_local = P.Tl * W
    N_total = T * W if seq_sharded else N_local * world

    rec = run_problem(rk, P, T, args, stream, ws, seq_sharded, count=True)
    check_guard(rec["guard_max_rel_err"], args.workload)
    ms_step = rec["ms_per_step"]
    value = N_total / (ms_step / 1e3)
    # the roofline's kernel durations: per-direction replays, or for short
    # steps the per-launch time of back-to-back launches (device_dir_ms)
    k_fwd_ms = rec.get("fwd_kernel_ms", rec["fwd_ms"])
    k_bwd_ms = rec.get("bwd_kernel_ms", rec["bwd_ms"])
    fwd_gbs = FWD_BYTES * N_local / (k_fwd_ms / 1e3) / 1e9
    bwd_gbs = BWD_BYTES * N_local / (k_bwd_ms / 1e3) / 1e9
    step_gbs = (FWD_BYTES + BWD_BYTES) * N_local / (ms_step / 1e3) / 1e9
    launches = rec.get("launches_per_step")

    # the same problem with slow decays lam ~ U(0.99, 1)
    slow = None
    if not args.no_slow:
        P.regen_lam(*LAM_SLOW, seed=77 + rank, stream=stream)
        srec = run_problem(rk, P, T, args, stream, ws, seq_sharded, steps=min(args.steps, 10))
        check_guard(srec["guard_max_rel_err"], args.workload + " slow decays")
        slow = dict(summarize(srec, N_total, N_local, peak), lam="U(0.99,1)")

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
            "median_ms_per_step": rec["median_ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong" if seq_sharded else "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": ("synthetic: lam~U(0.05,0.95), x,h0,dh~U(-1,1) (bench.hpp:134-143), generated on the host "
                     "(numpy PCG64, seeded) and copied to HBM; the CPU baseline / e2e leg / reference arm use "
                     "the same arrays"),
            "config": {
                "workload": wl["desc"],
                "T": T, "B": B, "D": D, "elements_per_step": N_total,
                "parallelism": ("sequence-sharded x%d (carry exchange: %s)" % (
                    world, "peer-memory mailboxes over NVLink" if rec.get("exchange") == "p2p" else "all-gather"))
                if seq_sharded
                else ("single GPU" if world == 1 else
                      "channel-sharded x%d (every rank an independent [T, B*D] block, no collective)" % world),
                "l2": "no flush: every tensor is %.0f MiB per GPU >> 126 MB L2" % (N_local * 4 / 2**20),
                "launch": "single GPU: the whole fwd+bwd step is one CUDA graph (captured once, replayed once per "
                          "timed step; fwd_ms/bwd_ms from per-direction graph replays outside the timed region); "
                          "sequence-sharded: eager (the exchange's epochs advance per step)",
                "timing": "CUDA events on the launching stream, barrier + synchronize around exactly `steps` "
                          "steps, max over ranks; value = elements / (total / steps)",
                "guard_max_rel_err": rec["guard_max_rel_err"],
            },
            "hbm_gbs": step_gbs,
            "pct_of_peak": 100.0 * step_gbs / peak,
            "kernels": {
                "fwd": {"ms": k_fwd_ms, "gbs": fwd_gbs, "bytes_per_element": FWD_BYTES,
                        "replay_ms": rec["fwd_ms"]},
                "bwd": {"ms": k_bwd_ms, "gbs": bwd_gbs, "bytes_per_element": BWD_BYTES,
                        "replay_ms": rec["bwd_ms"]},
                "timing": ("per-launch device time of 16 back-to-back launches per direction in one graph "
                           "(short step: a one-launch replay would charge ~4 us of graph launch to the kernel)"
                           if "fwd_kernel_ms" in rec else "per-direction graph replays"),
            },
            "roofline": {
                "bound": "hbm",
                "kernel": BWD_KERNEL_DESC[capi.scan_kernel_name(P.Tl, W, backward=True)],
                "achieved": bwd_gbs,
                "peak": peak,
                "peak_kind": peak_kind,
                "unit": "GB/s",
                "frac": bwd_gbs / peak,
                "traffic": traffic_from_profile(N_local),
                "algorithmic_bytes_per_launch": BWD_BYTES * N_local,
                "fwd": {"achieved": fwd_gbs, "frac": fwd_gbs / peak, "algorithmic_bytes_per_launch": FWD_BYTES * N_local},
            },
            "gpu_launches": (launches * args.steps) if launches is not None else None,
            "gpu_launches_method": "kernels of this repo per step counted with torch.profiler (CUPTI) over one "
                                   "untimed step, x steps",
            "clocks": rec["clocks"],
        }
        if slow is not None:
            result["slow_decay"] = slow
    P.free()
    torch.cuda.empty_cache()

    # C4 (BASELINE configs[3], the 1M-step workload) beside the C2 headline:
    # at N = 1 the single-GPU scan; at N > 1 also the sequence-sharded run over
    # all ranks and its strong-scaling speed-up over rank 0 alone.
    if args.workload == "c2" and not args.no_c4:
        c4 = c4_records(rk, args, stream, ws, peak)
        if rank == 0:
            result.update(c4)

    # the other BASELINE configs beside the C2 headline (1 GPU): C1, the C5
    # sweep and the C3 layer, so one default run records every config
    if args.workload == "c2" and world == 1 and not args.no_extra:
        extra = extra_records(rk, args, stream, ws, peak)
        if rank == 0:
            result.update(extra)

    # end to end through the public API with host buffers
    if not args.no_e2e and not seq_sharded:
        e2e = e2e_legs(rk, args, host, T, B, D)
        if rank == 0:
            result["e2e"] = e2e
    if rank == 0 and not args.no_cpu and world == 1:
        result["cpu_baseline"] = cpu_baseline_leg(args, host, T, B, D)
    del host
    if rank == 0:
        print(json.dumps(result), flush=True)
    rk.close()


def c4_records(rk, args, stream, ws, peak):
    """{"c4": ...} at N = 1; {"c4": ..., "c4_seq_sharded": ...} at N > 1."""
    import torch
    from paper_1709_04057_b200 import sharded
    wl = WORKLOADS["c4"]
    T, B, D = wl["T"], wl["B"], wl["D"]
    W = B * D
    out = {}
    # rank 0 alone: the 1-GPU C4 (the strong-scaling base)
    one = None
    if rk.rank == 0:
        one_rk = _Solo(rk)
        P = DeviceProblem(host_problem(T, B, D, SEED_C4), rk.dev, stream)
        rec = run_problem(one_rk, P, T, args, stream, ws, False)
        check_guard(rec["guard_max_rel_err"], "c4")
        one = summarize(rec, T * W, T * W, peak)
        if not args.no_slow:
            P.regen_lam(*LAM_SLOW, seed=78, stream=stream)
            srec = run_problem(one_rk, P, T, args, stream, ws, False, steps=min(args.steps, 10))
            check_guard(srec["guard_max_rel_err"], "c4 slow decays")
            one["slow_decay"] = dict(summarize(srec, T * W, T * W, peak), lam="U(0.99,1)")
        P.free()
        torch.cuda.empty_cache()
        out["c4"] = dict(one, workload=wl["desc"], n_gpus=1, T=T, W=W)
    rk.barrier()
    if rk.world > 1:
        r0, r1 = sharded.segment_bounds(T, rk.world, rk.rank)
        P = DeviceProblem(host_problem(T, B, D, SEED_C4, r0, r1), rk.dev, stream)
        rec = run_problem(rk, P, T, args, stream, ws, True, count=True)
        check_guard(rec["guard_max_rel_err"], "c4 sequence-sharded")
        rec_n = summarize(rec, T * W, P.Tl * W, peak)
        rec_n["exchange"] = rec.get("exchange")
        rec_n["launches_per_step_rank0"] = rec.get("launches_per_step")
        if not args.no_slow:
            P.regen_lam(*LAM_SLOW, seed=79 + rk.rank, stream=stream)
            srec = run_problem(rk, P, T, args, stream, ws, True, steps=min(args.steps, 10))
            check_guard(srec["guard_max_rel_err"], "c4 sequence-sharded slow decays")
            rec_n["slow_decay"] = dict(summarize(srec, T * W, P.Tl * W, peak), lam="U(0.99,1)")
        P.free()
        torch.cuda.empty_cache()
        if rk.rank == 0:
            rec_n.update(workload=wl["desc"] + " sequence-sharded", n_gpus=rk.world, T=T, W=W,
                         scaling="strong", n1_value=one["value"], n1_ms_per_step=one["ms_per_step"],
                         speedup=rec_n["value"] / one["value"])
            if "slow_decay" in rec_n and "slow_decay" in one:
                rec_n["slow_decay"]["speedup"] = rec_n["slow_decay"]["value"] / one["slow_decay"]["value"]
            out["c4_seq_sharded"] = rec_n
    return out


def extra_records(rk, args, stream, ws, peak):
    """{"c1": ..., "c5": ..., "c3": ...} on one GPU with bounded step counts
    (guards as in their own workloads; slow decays not repeated)."""
    import torch
    out = {}
    steps = min(args.steps, 20)
    solo = _Solo(rk)
    # C1 (configs[0]): the reference's correctness config
    wl = WORKLOADS["c1"]
    T, W = wl["T"], wl["B"] * wl["D"]
    P = DeviceProblem(host_problem(T, wl["B"], wl["D"], SEED_C2), rk.dev, stream)
    rec = run_problem(solo, P, T, args, stream, ws, False, steps=steps)
    check_guard(rec["guard_max_rel_err"], "c1")
    out["c1"] = dict(summarize(rec, T * W, T * W, peak), workload=wl["desc"], T=T, W=W)
    P.free()
    # C5 (configs[4]): 2^28 elements per (T, W) point
    pts, total = [], 0.0
    for k, (T, W) in enumerate(C5_POINTS):
        P = DeviceProblem(host_problem(T, 1, W, 5000 + k), rk.dev, stream)
        rec = run_problem(solo, P, T, args, stream, ws, False, steps=min(steps, 5))
        check_guard(rec["guard_max_rel_err"], f"c5 T={T} W={W}")
        pts.append(dict(summarize(rec, T * W, T * W, peak), T=T, W=W))
        total += rec["ms_per_step"]
        P.free()
        torch.cuda.empty_cache()
    n5 = sum(T * W for T, W in C5_POINTS)
    worst = min(pts, key=lambda p: p["frac_of_peak_per_gpu"])
    out["c5"] = {"value": n5 / (total / 1e3), "ms_per_step": total, "points": pts,
                 "worst_point": {"T": worst["T"], "W": worst["W"], "frac": worst["frac_of_peak_per_gpu"]},
                 "workload": "C5 fixed 2^28 elements per point, one fwd+bwd of every point per step (configs[4])"}
    # C3 (configs[2]): one GILR-LSTM layer fwd + bwd, tensor-core gate GEMMs + chained scans
    lr = layer_record(args, min(args.steps, 10), min(args.warmup, 3), False, False)
    out["c3"] = {k: lr[k] for k in ("value", "unit", "ms_per_step", "dtype", "events_per_s", "gemm_tflops_total",
                                    "gemm_share_of_step", "roofline")}
    out["c3"]["workload"] = lr["config"]["workload"]
    out["c3"]["guard_serial_vs_parallel"] = lr["config"]["guard_serial_vs_parallel"]
    torch.cuda.empty_cache()
    return out


class _Solo:
    """Ranks view of rank 0 alone (no collectives)."""

    def __init__(self, rk):
        self.world, self.rank, self.local, self.dev, self.share = 1, 0, rk.local, rk.dev, rk.share

    def barrier(self):
        pass

    def max(self, v):
        return v

    def gather(self, obj):
        return [obj]

    def bcast(self, obj):
        return obj


def e2e_legs(rk, args, host, T, B, D):
    """The metric end to end through the public API a reference user calls:
    ``linrec.scan`` / ``linrec.scan_backward`` on ordinary (pageable) numpy
    arrays, outputs freshly allocated per call (linrec_py.cpp:91-140) -- the
    headline e2e.  Secondary (N = 1): the host-pointer C ABI from pinned
    buffers.  At N > 1 every rank runs its own block concurrently (max over
    ranks)."""
    import numpy as np
    import torch
    from paper_1709_04057_b200 import capi, linrec

    lam, x, h0, dh = host
    W = B * D
    N = T * W
    steps = max(1, min(args.steps, args.e2e_steps))

    def step():
        h = linrec.scan(lam, x, h0)
        linrec.scan_backward(lam, h0, h, dh)

    step()  # warm: pipeline buffers, staging
    rk.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = rk.max((time.perf_counter() - t0) / steps)
    out = {
        "value": rk.world * N / dt,
        "unit": "elements/s",
        "ms_per_step": dt * 1e3,
        "steps": steps,
        # fwd: lam, x, h0 in / h out; bwd: lam, h0, h, dh in / dlam, dx, dh0 out (per rank x ranks)
        "h2d_bytes_per_step": rk.world * (4 * (2 * N + W) + 4 * (3 * N + W)),
        "d2h_bytes_per_step": rk.world * (4 * N + 4 * (2 * N + W)),
        "api": "paper_1709_04057_b200.linrec.scan + linrec.scan_backward (the reference's Python API, "
               "linrec_py.cpp:91-140) on pageable numpy arrays (staged through pinned bounce buffers by the library's "
               "copy threads), result arrays allocated per call (page-locked, from the library's caching host "
               "allocator)",
        "timing": "host wall clock around synchronous calls, max over ranks",
        "ranks": rk.world,
    }
    if rk.world == 1 and not args.no_pinned:
        pin = lambda s: torch.empty(s, dtype=torch.float32, pin_memory=True)  # noqa: E731
        shape = (T, B, D)
        pl, px, pdh, ph, pdl, pdx = (pin(shape) for _ in range(6))
        ph0, pdh0 = pin((B, D)), pin((B, D))
        for dst, src in ((pl, lam), (px, x), (pdh, dh), (ph0, h0)):
            dst.numpy()[...] = src
        p = lambda t: t.data_ptr()  # noqa: E731
        dev = rk.local

        def pstep():
            capi.scan_host(p(pl), p(px), p(ph0), p(ph), T, W, capi.PARALLEL, 4, dev)
            capi.scan_backward_host(p(pl), p(ph0), p(ph), p(pdh), p(pdl), p(pdx), p(pdh0), T, W,
                                    capi.PARALLEL, 4, dev)
        pstep()
        t0 = time.perf_counter()
        for _ in range(steps):
            pstep()
        dtp = (time.perf_counter() - t0) / steps
        out["pinned"] = {"value": N / dtp, "unit": "elements/s", "ms_per_step": dtp * 1e3, "steps": steps,
                         "api": "linrec_scan_host_f32 + linrec_scan_backward_host_f32 (C ABI) from pinned buffers"}
        del pl, px, pdh, ph, pdl, pdx, ph0, pdh0
    return out


def cpu_baseline_leg(args, host, T, B, D):
    """The reference's own CPU implementation (oracle/_ref, compiled from
    /root/reference with its -march=native flags where they fit this host) on
    the GPU arm's exact inputs, the whole C2 problem (no sampling): its
    scan_parallel + scan_backward(Parallel) with workers = all host cores, and
    the 1-core scan_serial + scan_backward(Serial); bench.hpp:93-107 protocol
    (median of reps, allocation inside the calls timed)."""
    try:
        from oracle.oracle import RefLib, ref_build
        ref_dir, march = ref_build()
        ref = RefLib(os.path.join(ref_dir, "liblinrec_ref.so"))
    except Exception as e:
        return {"value": None, "unit": "elements/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}
    lam, x, h0, dh = host
    cores = os.cpu_count() or 1
    n = T * B * D
    f, b = ref.bench_fwd_bwd(lam, x, h0, dh, cores, warmup=0, reps=args.cpu_reps)
    out = {
        "value": n / (f + b),
        "unit": "elements/s",
        "cores": cores,
        "kind": "reference",
        "sample": (f"the whole workload T={T} x B={B} x D={D} ({n} elements), the GPU arm's inputs: reference "
                   f"scan_parallel + scan_backward(ScanMode::Parallel), workers={cores}, median of "
                   f"{args.cpu_reps} rep(s)"),
        "cpu_model": cpu_model(),
        "build": f"oracle/_ref ({march}): recurrence.hpp + thread_pool.cpp compiled from /root/reference",
        "fwd_elements_per_s": n / f,
        "bwd_elements_per_s": n / b,
    }
    if not args.no_serial_cpu:
        fs, bs = ref.bench_serial(lam, x, h0, dh, warmup=0, reps=1)
        out["serial_1core"] = {"value": n / (fs + bs), "cores": 1,
                               "fwd_elements_per_s": n / fs, "bwd_elements_per_s": n / bs,
                               "sample": "same inputs: reference scan_serial + scan_backward(ScanMode::Serial)"}
    return out


# ---------------------------------------------------------------------------
# C5: the fixed-2^28-element sweep (BASELINE configs[4])
# ---------------------------------------------------------------------------
C5_POINTS = [(1 << 8, 1 << 20), (1 << 12, 1 << 16), (1 << 16, 1 << 12), (1 << 20, 1 << 8), (1 << 24, 1 << 4)]
C5_SEQ_SHARD_MAX_W = 256  # at N > 1: sequence sharding at W <= 256, channel sharding above


def run_c5(args):
    """Every (T, W) point at N = T*W = 2^28: one GPU, or N ranks sharing the
    fixed problem (strong scaling) -- channels split at large W (each rank a
    contiguous [T, W/N] block: no collective), the sequence at small W."""
    import torch
    from paper_1709_04057_b200 import capi, sharded
    rk = Ranks()
    stream = torch.cuda.Stream(device=rk.dev)
    ws = capi.Workspace(rk.local)
    peak, peak_kind = peaks()
    points = []
    total_ms = 0.0
    clocks = None
    launches = 0
    for k, (T, W) in enumerate(C5_POINTS):
        seq = rk.world > 1 and W <= C5_SEQ_SHARD_MAX_W
        if seq:
            r0, r1 = sharded.segment_bounds(T, rk.world, rk.rank)
            host = host_problem(T, 1, W, 5000 + k, r0, r1)
        elif rk.world > 1:
            c0, c1 = sharded.channel_shard(W, rk.world, rk.rank)
            host = host_problem(T, 1, c1 - c0, 5000 + 10 * k + rk.rank)
        else:
            host = host_problem(T, 1, W, 5000 + k)
        P = DeviceProblem(host, rk.dev, stream)
        del host
        rec = run_problem(rk, P, T, args, stream, ws, seq, count=True)
        check_guard(rec["guard_max_rel_err"], f"c5 T={T} W={W}")
        rec_s = summarize(rec, T * W, P.Tl * P.W, peak)
        rec_s.update(T=T, W=W, sharding=("sequence" if seq else "channel" if rk.world > 1 else "none"))
        points.append(rec_s)
        total_ms += rec["ms_per_step"]
        launches += rec.get("launches_per_step") or 0
        clocks = rec["clocks"]
        P.free()
        torch.cuda.empty_cache()
    if rk.rank == 0:
        n_total = sum(T * W for T, W in C5_POINTS)
        best = max(points, key=lambda p: p["frac_of_peak_per_gpu"])
        worst = min(points, key=lambda p: p["frac_of_peak_per_gpu"])
        print(json.dumps({
            "metric": METRIC,
            "value": n_total / (total_ms / 1e3),
            "unit": "elements/s",
            "n_gpus": rk.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic: lam~U(0.05,0.95), x,h0,dh~U(-1,1), host-generated",
            "config": {"workload": "C5 fixed 2^28 elements per point, (T, W) in " +
                       ", ".join(f"(2^{T.bit_length() - 1}, 2^{W.bit_length() - 1})" for T, W in C5_POINTS) +
                       " (BASELINE configs[4]); a step = one fwd+bwd of every point",
                       "parallelism": "single GPU" if rk.world == 1 else
                       f"x{rk.world}: sequence-sharded at W <= {C5_SEQ_SHARD_MAX_W}, channel-sharded above",
                       "l2": "no flush: every tensor is 1 GiB (/N per GPU)"},
            "points": points,
            "roofline": {"bound": "hbm", "kernel": "fwd+bwd chained scans per point", "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "achieved": best["hbm_gbs_per_gpu"], "frac": best["frac_of_peak_per_gpu"],
                         "worst_point": {"T": worst["T"], "W": worst["W"], "frac": worst["frac_of_peak_per_gpu"]},
                         "traffic": None},
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
        }), flush=True)
    rk.close()


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation through its public
# Python API (oracle/_ref/linrec*.so = proj/bindings/linrec_py.cpp compiled
# from /root/reference), on this host's cores, on the SAME config and inputs
# as our arm's rank 0 (no sampling).
# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    try:
        from oracle.oracle import load_reference_module, ref_build
        ref_dir, march = ref_build()
        ref = load_reference_module(ref_dir)
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {e}"}))
        return
    cores = os.cpu_count() or 1
    if args.workload == "c5":
        points = C5_POINTS
        seeds = [5000 + k for k in range(len(points))]
        desc = "C5 fixed 2^28 elements per point (BASELINE configs[4])"
        shapes = [(T, 1, W) for T, W in points]
    else:
        wl = WORKLOADS[args.workload]
        shapes = [(wl["T"], wl["B"], wl["D"])]
        seeds = [SEED_C4 if args.workload == "c4" else SEED_C2]
        desc = wl["desc"]
    probs = [host_problem(*shp, seed) for shp, seed in zip(shapes, seeds)]

    def step():
        for lam, x, h0, dh in probs:
            h = ref.scan(lam, x, h0, workers=cores)
            ref.scan_backward(lam, h0, h, dh, workers=cores)

    steps, warmup = args.steps, args.warmup
    if args.workload == "c5":  # 5 x 2^28 elements per step on the host: bounded
        steps, warmup = min(steps, 2), min(warmup, 1)
    for _ in range(warmup):
        step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    n = sum(T * B * D for T, B, D in shapes)
    value = n / (ms / 1e3)
    sample = (f"the whole workload ({n} elements per step, the same seeded inputs as our arm's rank 0): "
              f"linrec.scan + linrec.scan_backward (reference pybind11 API, numpy in/out), workers={cores}, "
              f"build {march}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms,
        "median_ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: lam~U(0.05,0.95), x,h0,dh~U(-1,1), host-generated (numpy PCG64, seeded)",
        "config": {"workload": desc, "shapes": shapes, "sampled": False},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model()},
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
        "scan_bwd_cell": ("byte", 20 * E),       # f, dh, o (dc = dh * o fused in), c in; G out (dlam: in dpre)
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


CUBLAS_TF32_TFLOPS = 755.0  # measured: torch.matmul fp32 with allow_tf32, 262144 x 2048 x 1024 (C3's gate GEMM shape)


def tensor_peak():
    """Dense TF32 tensor-core peak for the roofline: the nominal 1.1 PFLOP/s
    of B200_PROFILING.md.  MEASURED_PEAKS.json has no TF32 figure, and half of
    its measured bf16 rate (cuBLAS) is no upper bound here: the 3xTF32 GEMMs
    issue MMAs at ~900 TF/s with the split disabled."""
    return 1100.0, "nominal dense TF32 (B200_PROFILING.md); no measured TF32 peak exists"


def run_layer(args):
    world, rank, local = dist_env()
    if world > 1:
        raise SystemExit("c3 is a single-GPU workload (the layer shards like C2 over channels: run replicas)")
    result = layer_record(args, args.steps, args.warmup, not args.no_e2e, not args.no_cpu)
    print(json.dumps(result), flush=True)


def layer_record(args, steps, warmup, with_e2e, with_cpu):
    """One GILR-LSTM layer fwd + bwd at C3 (BASELINE configs[2]): the timed
    record (per-stage GEMM / scan rates, roofline, guard)."""
    import torch
    from paper_1709_04057_b200 import layers as L

    world, rank, local = dist_env()
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

        for _ in range(warmup):
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
        for _ in range(steps):
            step()
        end.record(stream)
        torch.cuda.synchronize(dev)
    stages = L.profile_end()
    ms = start.elapsed_time(end) / steps
    E = T * b * n
    work = layer_stage_work(T, b, m, n)
    hbm, hbm_kind = peaks()
    tpk, tpk_kind = tensor_peak()
    st_out, best = {}, None
    for name, (tot, cnt) in stages.items():
        avg = tot / steps
        rec = {"ms": avg, "launch_sets_per_step": cnt / steps}
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
        "steps": steps,
        "warmup": warmup,
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
            # cuBLAS's own TF32 GEMM on this pool's B200s (scripts/dev/cublas_tf32.py: 703-755 TF/s
            # at 8192^3 and the C3 shapes): the practical ceiling of the MMA issue rate
            "cublas_tf32_tflops": CUBLAS_TF32_TFLOPS,
            "mma_issue_frac_of_cublas": (3 if prec == "fp32" else 1) * achieved / CUBLAS_TF32_TFLOPS,
            "effective_peak_for_precision": tpk / (3 if prec == "fp32" else 1),
            "traffic": None,
            "algorithmic_flops_per_launch": bflop,
        },
        "gpu_launches": None,
        "clocks": clocks.summary(),
    }
    # kernels per step counted on the device with torch.profiler (untimed pass)
    counted = count_our_kernels(step)
    result["gpu_launches"] = (counted * steps if counted is not None
                              else sum(round(v["launch_sets_per_step"]) for v in st_out.values()) * steps)
    result["gpu_launches_method"] = ("kernels of this repo per step counted with torch.profiler (CUPTI) over one "
                                     "untimed step, x steps" if counted is not None else "stage call count")
    del cache, grads
    torch.cuda.empty_cache()
    if with_e2e:
        result["e2e"] = layer_e2e(args, p, T, b, m, n, dev)
    if with_cpu:
        result["cpu_baseline"] = layer_cpu_baseline(args, m, n, b)
    return result


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


def relaunch(args):
    """--gpus N without torchrun: re-exec this script under
    torch.distributed.run, one rank per GPU (the driver's own launch form)."""
    import subprocess
    import socket
    if os.environ.get("LINREC_BENCH_SHARE_GPU") != "1" and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} GPU(s) visible "
                             "(LINREC_BENCH_SHARE_GPU=1 lets ranks share GPUs, for tests)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["c5"], default="c2")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-reps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pinned", action="store_true", help="skip the secondary pinned-buffer e2e figure")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-serial-cpu", action="store_true", help="skip the 1-core reference row")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 records beside the C2 headline")
    ap.add_argument("--no-slow", action="store_true", help="skip the lam~U(0.99,1) re-runs")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the C1 / C5 / C3 records beside the C2 headline (1 GPU)")
    ap.add_argument("--precision", choices=["fp32", "tf32"], default="fp32", help="c3 GEMM precision")
    ap.add_argument("--layer-cpu-rows", type=int, default=16)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    if args.workload == "c3":
        run_reference_layer(args) if args.impl == "reference" else run_layer(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
