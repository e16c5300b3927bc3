"""Tuning sweep of the chained-scan kernels on the C2 workload (GPU only).

Times fwd and bwd for each TMA configuration (LINREC_TMA_FWD / LINREC_TMA_BWD
= "R,STAGES") and for the register kernels, checking each against the serial
kernel.  Prints one JSON line per configuration.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_04057_b200 import capi  # noqa: E402

T, B, D = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (65536, 8, 1024))]
W = B * D
N = T * W
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
lam = torch.empty(T, W, device=dev).uniform_(0.05, 0.95, generator=g)
x = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h0 = torch.empty(W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(T, W, device=dev).uniform_(-1, 1, generator=g)
h = torch.empty_like(lam)
dlam = torch.empty_like(lam)
dx = torch.empty_like(lam)
dh0 = torch.empty_like(h0)
ref_h = torch.empty_like(lam)
st = torch.cuda.current_stream().cuda_stream
ws = capi.Workspace(0)
p = lambda t: t.data_ptr()  # noqa: E731
capi.scan(p(lam), p(x), p(h0), p(ref_h), T, W, capi.SERIAL, 4, None, st)
ref_dx = torch.empty_like(lam)
ref_dlam = torch.empty_like(lam)
capi.scan_backward(p(lam), p(h0), p(ref_h), p(dh), p(ref_dlam), p(ref_dx), p(dh0), T, W, capi.SERIAL, 4, None, st)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def fwd():
    capi.scan(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, ws.handle, st)


def bwd():
    capi.scan_backward(p(lam), p(h0), p(ref_h), p(dh), p(dlam), p(dx), p(dh0), T, W, capi.PARALLEL, 4, ws.handle, st)


def err(a, b):
    return ((a - b).abs().max() / b.abs().max()).item()


peak = 6555.2
try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    _h = None

configs = [] if os.environ.get("TUNE_NO_REGISTER") else [("register", None, None)]
configs += [("tma", f, None) for f in os.environ.get("TUNE_FWD", "8,2,8;8,3,8;12,2,8;16,2,4;16,3,4;16,1,8;4,3,8").split(";")]
configs += [("tma", None, b) for b in os.environ.get("TUNE_BWD", "8,2,8;6,2,8;12,1,8;8,2,4;12,2,4;4,3,8").split(";")]
for kind, fc, bc in configs:
    capi.set_kernel_policy(capi.KERNEL_REGISTER if kind == "register" else capi.KERNEL_AUTO)
    for k, v in (("LINREC_TMA_FWD", fc), ("LINREC_TMA_BWD", bc)):
        if v:
            os.environ[k] = v
        else:
            os.environ.pop(k, None)
    rec = {"kind": kind, "fwd_cfg": fc, "bwd_cfg": bc, "T": T, "W": W}
    print("start", kind, fc, bc, file=sys.stderr, flush=True)
    if kind == "register" or fc:
        ms = timeit(fwd)
        rec.update(fwd_ms=ms, fwd_gbs=12 * N / ms / 1e6, fwd_frac=12 * N / ms / 1e6 / peak, fwd_err=err(h, ref_h))
    if kind == "register" or bc:
        ms = timeit(bwd)
        rec.update(bwd_ms=ms, bwd_gbs=20 * N / ms / 1e6, bwd_frac=20 * N / ms / 1e6 / peak,
                   bwd_err=max(err(dx, ref_dx), err(dlam, ref_dlam)))
    if _h is not None:
        rec["sm_mhz"] = pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM)
    rec["lib"] = os.path.basename(capi.LIB_PATH)
    print(json.dumps(rec), flush=True)
