"""Stress the parallel scans at one shape: `iters` fwd+bwd launches on fresh
random data, each checked against the per-channel serial kernels (max
normwise error, the bench guard's metric).  Prints the failures.
Usage: stress_scan.py T W iters [seed] [graph]  (graph=1: the parallel fwd+bwd
captured once into a CUDA graph on a side stream and replayed, as bench.py)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402

T, W, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 0
use_graph = len(sys.argv) > 5 and sys.argv[5] == "1"
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(seed)
st = torch.cuda.current_stream().cuda_stream
ws = capi.Workspace(0)
p = lambda t: t.data_ptr()  # noqa: E731


def rel(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1.0)).item()


lam = torch.empty(T, W, device=dev)
x, dh, h0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty(W, device=dev)
h, dl, dx, d0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
hs, dls, dxs, d0s = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(h0)
side = torch.cuda.Stream()
sst = side.cuda_stream


def par(s):
    capi.scan(p(lam), p(x), p(h0), p(h), T, W, capi.PARALLEL, 4, ws.handle, s)
    capi.scan_backward(p(lam), p(h0), p(h), p(dh), p(dl), p(dx), p(d0), T, W, capi.PARALLEL, 4, ws.handle, s)


graph = None
if use_graph:
    par(sst)
    side.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        par(sst)
bad = 0
for it in range(iters):
    lam.uniform_(0.05, 0.95, generator=g)
    x.uniform_(-1, 1, generator=g)
    dh.uniform_(-1, 1, generator=g)
    h0.uniform_(-1, 1, generator=g)
    if graph is not None:
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            graph.replay()
            graph.replay()
        torch.cuda.synchronize()
    else:
        par(st)
    capi.scan(p(lam), p(x), p(h0), p(hs), T, W, capi.SERIAL, 4, None, st)
    capi.scan_backward(p(lam), p(h0), p(hs), p(dh), p(dls), p(dxs), p(d0s), T, W, capi.SERIAL, 4, None, st)
    torch.cuda.synchronize()
    e = max(rel(h, hs), rel(dl, dls), rel(dx, dxs), rel(d0, d0s))
    if not e <= 1e-5:
        bad += 1
        eh, ed = rel(h, hs), rel(dx, dxs)
        rows = ((h - hs).abs() > 1e-3).any(dim=1).nonzero().flatten()
        cols = ((h - hs).abs() > 1e-3).any(dim=0).nonzero().flatten()
        print(f"iter {it}: err {e:.3e} (h {eh:.3e}, dx {ed:.3e}); bad h rows {rows[:8].tolist()}.. "
              f"({len(rows)}), cols {cols[:8].tolist()}.. ({len(cols)})", flush=True)
print(f"T={T} W={W} seed={seed}: {bad} of {iters} iterations failed", flush=True)
