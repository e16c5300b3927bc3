"""Per-rank work of the sequence-sharded C4 step at N ranks, on one GPU:
segment scan (zero carry) + the carry fold + fix-up, forward and backward,
for rank 1 of N (a middle rank: receives forward and backward carries).
The peer exchange itself is replaced by a local fold (world=1 plumbing), so
this times everything but the NVLink latency.  Usage: rank_work.py N [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1709_04057_b200 import capi  # noqa: E402
from paper_1709_04057_b200.sharded import segment_rows  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
T, W = 1 << 20, 128
Tl = segment_rows(T, N, 1)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
lam = torch.empty(Tl, W, device=dev).uniform_(0.05, 0.95, generator=g)
x = torch.empty(Tl, W, device=dev).uniform_(-1, 1, generator=g)
dh = torch.empty(Tl, W, device=dev).uniform_(-1, 1, generator=g)
h, dlam, dx = torch.empty_like(lam), torch.empty_like(lam), torch.empty_like(lam)
dh0 = torch.empty(W, device=dev)
hprev = torch.empty(W, device=dev).uniform_(-1, 1, generator=g)
ones = torch.ones(W, device=dev)
nf, nb = capi.segment_prod_rows(Tl, W, False), capi.segment_prod_rows(Tl, W, True)
rf, rb = capi.segment_tile_rows(Tl, W, False), capi.segment_tile_rows(Tl, W, True)
spf, spb = torch.empty(nf, W, device=dev), torch.empty(nb, W, device=dev)
agg = torch.empty(2, W, device=dev)
aggs = torch.empty(N, 2, W, device=dev).uniform_(0, 0.5, generator=g)
c_in, y_in = torch.empty(W, device=dev), torch.empty(W, device=dev)
ws = capi.Workspace(0)
st = torch.cuda.current_stream().cuda_stream
p = lambda t: t.data_ptr()  # noqa: E731


def fwd():
    capi.segment_scan(p(lam), p(x), None, p(h), p(spf), p(agg), Tl, W, 4, ws.handle, st)
    capi.compose_carries(p(aggs), 0, 1, 1, None, p(c_in), W, 4, st)
    capi.segment_fixup(p(lam), p(h), p(spf), p(c_in), Tl, W, rf, 4, st)


def bwd():
    capi.segment_scan_backward(p(lam), p(hprev), p(h), p(dh), p(ones), p(dlam), p(dx), p(dh0), p(spb), p(agg), Tl, W,
                               4, ws.handle, st)
    capi.compose_carries(p(aggs), N - 1, 1, -1, None, p(y_in), W, 4, st)
    capi.segment_fixup_backward(p(lam), p(hprev), p(h), p(ones), p(spb), p(y_in), p(dlam), p(dx), Tl, W, rb, 4, st)


for _ in range(5):
    fwd()
    bwd()
torch.cuda.synchronize()
# the same launches replayed from CUDA graphs: GPU time without host gaps
s2 = torch.cuda.Stream()
st_saved = st
with torch.cuda.stream(s2):
    st = s2.cuda_stream
    gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    fwd(); bwd()  # warm the workspace on this stream
    torch.cuda.synchronize()
    with torch.cuda.graph(gf, stream=s2):
        fwd()
    with torch.cuda.graph(gb, stream=s2):
        bwd()
torch.cuda.synchronize()
st = st_saved
e3 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
gtf = gtb = 0.0
for _ in range(reps):
    e3[0].record()
    gf.replay()
    e3[1].record()
    gb.replay()
    e3[2].record()
    torch.cuda.synchronize()
    gtf += e3[0].elapsed_time(e3[1])
    gtb += e3[1].elapsed_time(e3[2])
print(f"N={N} graph-replayed: fwd {gtf / reps * 1e3:.1f} us  bwd {gtb / reps * 1e3:.1f} us", flush=True)
# the whole step (fwd + bwd) as ONE graph, as bench.py times a single-GPU step
with torch.cuda.stream(s2):
    st = s2.cuda_stream
    gstep = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gstep, stream=s2):
        fwd()
        bwd()
torch.cuda.synchronize()
st = st_saved
e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e2[0].record()
for _ in range(reps):
    gstep.replay()
e2[1].record()
torch.cuda.synchronize()
print(f"N={N} one-graph step: {e2[0].elapsed_time(e2[1]) / reps * 1e3:.1f} us per rank-step "
      f"(7x over the 1-GPU C4 step needs <= {721.3 / 7:.0f} us)", flush=True)
# the peer-exchange path has no compose launch: the fix-up CTAs fold the
# peers' aggregates from their mailboxes (p2p_impl.cuh::compose_chunk); here
# c_in / y_in stay as computed above
with torch.cuda.stream(s2):
    st = s2.cuda_stream
    gstep2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gstep2, stream=s2):
        capi.segment_scan(p(lam), p(x), None, p(h), p(spf), p(agg), Tl, W, 4, ws.handle, st)
        capi.segment_fixup(p(lam), p(h), p(spf), p(c_in), Tl, W, rf, 4, st)
        capi.segment_scan_backward(p(lam), p(hprev), p(h), p(dh), p(ones), p(dlam), p(dx), p(dh0), p(spb), p(agg),
                                   Tl, W, 4, ws.handle, st)
        capi.segment_fixup_backward(p(lam), p(hprev), p(h), p(ones), p(spb), p(y_in), p(dlam), p(dx), Tl, W, rb, 4,
                                    st)
torch.cuda.synchronize()
st = st_saved
e2[0].record()
for _ in range(reps):
    gstep2.replay()
e2[1].record()
torch.cuda.synchronize()
print(f"N={N} one-graph step without the compose launches (as the peer-exchange path): "
      f"{e2[0].elapsed_time(e2[1]) / reps * 1e3:.1f} us per rank-step", flush=True)
# per kernel (each launch its own graph, replayed back to back in step order)
parts = {
    "fwd scan": lambda: capi.segment_scan(p(lam), p(x), None, p(h), p(spf), p(agg), Tl, W, 4, ws.handle, st),
    "fwd compose": lambda: capi.compose_carries(p(aggs), 0, 1, 1, None, p(c_in), W, 4, st),
    "fwd fixup": lambda: capi.segment_fixup(p(lam), p(h), p(spf), p(c_in), Tl, W, rf, 4, st),
    "bwd scan": lambda: capi.segment_scan_backward(p(lam), p(hprev), p(h), p(dh), p(ones), p(dlam), p(dx), p(dh0),
                                                   p(spb), p(agg), Tl, W, 4, ws.handle, st),
    "bwd compose": lambda: capi.compose_carries(p(aggs), N - 1, 1, -1, None, p(y_in), W, 4, st),
    "bwd fixup": lambda: capi.segment_fixup_backward(p(lam), p(hprev), p(h), p(ones), p(spb), p(y_in), p(dlam),
                                                     p(dx), Tl, W, rb, 4, st),
}
graphs = {}
with torch.cuda.stream(s2):
    st = s2.cuda_stream
    for name, fn in parts.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s2):
            fn()
        graphs[name] = g
torch.cuda.synchronize()
st = st_saved
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(parts) + 1)]
acc = dict.fromkeys(parts, 0.0)
for _ in range(reps):
    evs[0].record()
    for i, name in enumerate(parts):
        graphs[name].replay()
        evs[i + 1].record()
    torch.cuda.synchronize()
    for i, name in enumerate(parts):
        acc[name] += evs[i].elapsed_time(evs[i + 1])
print("  per kernel: " + ", ".join(f"{k} {v / reps * 1e3:.1f}" for k, v in acc.items()) + " us", flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf = tb = 0.0
for _ in range(reps):
    ev[0].record()
    fwd()
    ev[1].record()
    bwd()
    ev[2].record()
    torch.cuda.synchronize()
    tf += ev[0].elapsed_time(ev[1])
    tb += ev[1].elapsed_time(ev[2])
tf, tb = tf / reps * 1e3, tb / reps * 1e3
ideal = 32 * Tl * W / 6.535e12 * 1e6
print(f"N={N} rows={Tl} fwd {tf:.1f} us  bwd {tb:.1f} us  total {tf + tb:.1f} us  "
      f"(ideal {ideal:.1f} us at measured peak; 1-GPU C4 step / 7 = 111 us)", flush=True)
