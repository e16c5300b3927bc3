"""Multi-GPU sharding of the linear recurrence.

* Channel sharding -- channels are independent (recurrence.hpp:109): every
  rank owns a [T, W/N] block and calls the single-GPU scans; there is no
  collective on the data path (`channel_shard`).
* Sequence sharding -- T is split into contiguous segments, one per rank
  (`segment_bounds`).  Per direction each rank runs ONE zero-carry chained scan
  of its segment (12 / 20 B/element), the ranks exchange a 2*W-value carry
  and a fix-up kernel adds the carry's decaying contribution to the leading
  tiles of the segment (include/linrec_cuda.h, csrc/segment.cu).  The
  exchange is the only inter-GPU traffic: 2*W*4 bytes per rank per direction
  (1 KiB at W = 128).  By default it goes over peer memory (``PeerMailboxes``,
  csrc/p2p.cu): each rank stores its aggregate straight into the consumers'
  mailboxes over NVLink and raises a release flag that their fold kernel
  acquires -- no collective launch, a few microseconds instead of an NCCL
  all-gather's ~15.  Ranks on different nodes (no CUDA IPC) fall back to the
  all-gather.

The orchestration is written against a small backend interface so that the
same code drives the CUDA kernels (``CudaBackend``, NCCL) and, in the CPU test
suite, a reference backend over gloo.  The product backend is the CUDA one;
this module has no CPU compute path.
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist

from . import capi


def segment_bounds(T: int, world: int, rank: int):
    """Rows [start, end) of rank's segment: contiguous, sizes differing by at
    most one, longer segments first (the reference's plan_chunks rule,
    recurrence.hpp:61-80, applied to ranks)."""
    base, rem = divmod(T, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def segment_rows(T: int, world: int, rank: int) -> int:
    s, e = segment_bounds(T, world, rank)
    return e - s


def channel_shard(W: int, world: int, rank: int):
    """Channels [start, end) owned by rank under channel sharding: contiguous
    blocks, multiples of 4 channels when W allows (16-byte rows for the
    vector kernels), longer blocks first (linrec_column_block)."""
    unit = 4 if W % 4 == 0 else 1
    s, e = segment_bounds(W // unit, world, rank)
    return s * unit, e * unit


def _host_arrays(*arrays):
    import numpy as np
    out = []
    dt = None
    for a in arrays:
        if a is None:
            out.append(None)
            continue
        a = np.ascontiguousarray(a)
        if dt is None:
            dt = a.dtype
            if dt not in (np.float32, np.float64):
                raise TypeError("decays must be float32 or float64")
        elif a.dtype != dt:
            raise TypeError("all arrays must share the decays dtype")
        out.append(a)
    return out, dt


def _ptr(a):
    return None if a is None else a.ctypes.data


def _mode(mode):
    if mode not in ("parallel", "serial"):
        raise ValueError(f"unknown mode '{mode}' (expected 'serial' or 'parallel')")
    return capi.SERIAL if mode == "serial" else capi.PARALLEL


def channel_sharded_scan(decays, impulses, initial=None, *, devices=None, mode="parallel"):
    """scan (recurrence.hpp:255-263) of host [T, b, n] arrays with the channels
    split over `devices` (default: every visible GPU) -- one host thread per
    GPU, each staging its column block with 2-D copies; no communication
    (channels are independent, recurrence.hpp:109).  numpy in, numpy out."""
    import numpy as np
    (lam, x, h0), dt = _host_arrays(decays, impulses, initial)
    if lam.ndim != 3:
        raise ValueError("decays must have shape [T, batch, features]")
    if lam.shape != x.shape:
        raise RuntimeError(f"recurrence: shape mismatch, {list(lam.shape)} vs {list(x.shape)}")
    if h0 is not None and h0.shape != lam.shape[1:]:
        raise RuntimeError(f"recurrence: initial state {list(h0.shape)} does not match {list(lam.shape[1:])}")
    T, W = lam.shape[0], lam.shape[1] * lam.shape[2]
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    h = np.empty_like(lam)
    capi.scan_host_multi(_ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, W, devices, _mode(mode), dt.itemsize)
    return h


def channel_sharded_scan_backward(decays, initial, h, d_h, *, devices=None, mode="parallel"):
    """scan_backward (recurrence.hpp:352-363) of host arrays, channels split
    over `devices` like channel_sharded_scan: (d_decays, d_impulses, d_initial)."""
    import numpy as np
    (lam, h0, hh, dh), dt = _host_arrays(decays, initial, h, d_h)
    if lam.ndim != 3:
        raise ValueError("decays must have shape [T, batch, features]")
    for a, n in ((hh, "h"), (dh, "d_h")):
        if a.shape != lam.shape:
            raise RuntimeError(f"scan_backward({n}): shape mismatch, {list(lam.shape)} vs {list(a.shape)}")
    if h0 is not None and h0.shape != lam.shape[1:]:
        raise RuntimeError(f"recurrence: initial state {list(h0.shape)} does not match {list(lam.shape[1:])}")
    T, W = lam.shape[0], lam.shape[1] * lam.shape[2]
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    dlam, dx = np.empty_like(lam), np.empty_like(lam)
    dh0 = np.empty(lam.shape[1:], dtype=dt)
    capi.scan_backward_host_multi(_ptr(lam), _ptr(h0), _ptr(hh), _ptr(dh), _ptr(dlam), _ptr(dx), _ptr(dh0), T, W,
                                  devices, _mode(mode), dt.itemsize)
    return dlam, dx, dh0


class ChannelShardedScan:
    """One process per GPU: rank r scans its channel block (channel_shard) of
    the caller's full host arrays on its own device and writes those columns
    of the outputs; `gather=True` all-gathers the other ranks' columns over
    the process group (host tensors), so every rank ends with the full
    result.  No collective on the data path otherwise."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = torch.cuda.current_device() if device is None else device

    def columns(self, W):
        return channel_shard(W, self.world, self.rank)

    def _gather(self, arr, W):
        if self.world == 1:
            return
        import numpy as np
        T = arr.shape[0]
        flat = arr.reshape(T, W)
        blocks = [channel_shard(W, self.world, q) for q in range(self.world)]
        wmax = max(e - s for s, e in blocks)  # all_gather needs equal sizes: pad to the widest block
        s0, e0 = blocks[self.rank]
        mine = torch.zeros(T, wmax, dtype=torch.from_numpy(flat[:0, :0]).dtype)
        mine[:, :e0 - s0] = torch.from_numpy(np.ascontiguousarray(flat[:, s0:e0]))
        parts = [torch.empty_like(mine) for _ in blocks]
        dist.all_gather(parts, mine, group=self.group)
        for (s, e), part in zip(blocks, parts):
            flat[:, s:e] = part[:, :e - s].numpy()

    def scan(self, decays, impulses, initial=None, *, mode="parallel", gather=False):
        import numpy as np
        (lam, x, h0), dt = _host_arrays(decays, impulses, initial)
        T, W = lam.shape[0], lam.shape[1] * lam.shape[2]
        c0, c1 = self.columns(W)
        h = np.zeros_like(lam)
        if c0 < c1:
            capi.scan_host_columns(_ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, W, c0, c1, _mode(mode), dt.itemsize,
                                   self.device)
        if gather:
            self._gather(h, W)
        return h

    def scan_backward(self, decays, initial, h, d_h, *, mode="parallel", gather=False):
        import numpy as np
        (lam, h0, hh, dh), dt = _host_arrays(decays, initial, h, d_h)
        T, W = lam.shape[0], lam.shape[1] * lam.shape[2]
        c0, c1 = self.columns(W)
        dlam, dx = np.zeros_like(lam), np.zeros_like(lam)
        dh0 = np.zeros(lam.shape[1:], dtype=dt)
        if c0 < c1:
            capi.scan_backward_host_columns(_ptr(lam), _ptr(h0), _ptr(hh), _ptr(dh), _ptr(dlam), _ptr(dx),
                                            _ptr(dh0), T, W, c0, c1, _mode(mode), dt.itemsize, self.device)
        if gather:
            for a in (dlam, dx):
                self._gather(a, W)
            self._gather(dh0.reshape(1, -1), W)
        return dlam, dx, dh0


class CudaBackend:
    """Primitive operations of the sharded scan on the sm_100a kernels."""

    def __init__(self, ws=None, stream=None):
        self.ws = ws
        self.stream = stream

    def _st(self):
        s = self.stream if self.stream is not None else torch.cuda.current_stream()
        return s.cuda_stream

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def tile_rows(self, T, W, backward):
        return capi.segment_tile_rows(T, W, backward)

    def prod_rows(self, T, W, backward):
        return capi.segment_prod_rows(T, W, backward)

    def segment_scan(self, lam, x, h0, h, seg_prod, agg, T, W):
        capi.segment_scan(lam.data_ptr(), x.data_ptr(), self._p(h0), h.data_ptr(), seg_prod.data_ptr(),
                          agg.data_ptr(), T, W, 4, None if self.ws is None else self.ws.handle, self._st())

    def segment_scan_backward(self, lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W):
        capi.segment_scan_backward(lam.data_ptr(), self._p(hprev), h.data_ptr(), dh.data_ptr(),
                                   self._p(lam_next), dlam.data_ptr(), dx.data_ptr(), dh0.data_ptr(),
                                   seg_prod.data_ptr(), agg.data_ptr(), T, W, 4,
                                   None if self.ws is None else self.ws.handle, self._st())

    def compose(self, aggs, first, last, step, seed, out, W):
        capi.compose_carries(aggs.data_ptr(), first, last, step, self._p(seed), out.data_ptr(), W, 4, self._st())

    def fixup(self, lam, h, seg_prod, c_in, T, W, rows):
        capi.segment_fixup(lam.data_ptr(), h.data_ptr(), seg_prod.data_ptr(), self._p(c_in), T, W, rows, 4,
                           self._st())

    # the exchange fused into the stitch kernels (PeerMailboxes.exchange)
    def segment_scan_exchange(self, lam, x, h0, h, seg_prod, agg, T, W, ex):
        capi.segment_scan_exchange(lam.data_ptr(), x.data_ptr(), self._p(h0), h.data_ptr(), seg_prod.data_ptr(),
                                   agg.data_ptr(), T, W, ex, None if self.ws is None else self.ws.handle, self._st())

    def segment_scan_backward_exchange(self, lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ex):
        capi.segment_scan_backward_exchange(lam.data_ptr(), self._p(hprev), h.data_ptr(), dh.data_ptr(),
                                            self._p(lam_next), dlam.data_ptr(), dx.data_ptr(), dh0.data_ptr(),
                                            seg_prod.data_ptr(), agg.data_ptr(), T, W, ex,
                                            None if self.ws is None else self.ws.handle, self._st())

    def fixup_exchange(self, lam, h, seg_prod, c_in, T, W, rows, ex):
        capi.segment_fixup_exchange(lam.data_ptr(), h.data_ptr(), seg_prod.data_ptr(), c_in.data_ptr(), T, W, rows,
                                    ex, self._st())

    def fixup_backward_exchange(self, lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, rows, ex):
        capi.segment_fixup_backward_exchange(lam.data_ptr(), self._p(hprev), h.data_ptr(), self._p(lam_next),
                                             seg_prod.data_ptr(), y_in.data_ptr(), dlam.data_ptr(), dx.data_ptr(),
                                             T, W, rows, ex, self._st())

    def fixup_backward(self, lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, rows):
        capi.segment_fixup_backward(lam.data_ptr(), self._p(hprev), h.data_ptr(), self._p(lam_next),
                                    seg_prod.data_ptr(), self._p(y_in), dlam.data_ptr(), dx.data_ptr(), T, W,
                                    rows, 4, self._st())


class PeerMailboxes:
    """One CUDA-IPC mailbox per rank (csrc/p2p.cu); every rank maps every
    peer's.  Handles travel once through the process group."""

    def __init__(self, W, group, device):
        import ctypes as C
        lib = capi.lib
        self.group, self.W = group, W
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        nbytes = lib.linrec_p2p_mailbox_bytes(W, self.world)
        own, handle = C.c_void_p(), C.create_string_buffer(64)
        # no rank raises before the collectives: a failure is recorded
        # (self.error) and every rank still takes part, so the caller can
        # agree on a fallback (SequenceShardedScan, exchange="auto")
        self.error = None
        rc = lib.linrec_ipc_alloc(nbytes, C.byref(own), handle)
        if rc != capi.OK:
            self.error = capi.LinrecError(rc, lib.linrec_last_error().decode())
        self.own = own.value if rc == capi.OK else None
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw if rc == capi.OK else None, group=group)
        self.opened, ptrs = [], []
        for q, h in enumerate(handles):
            if q == self.rank:
                ptrs.append(self.own or 0)
                continue
            p = C.c_void_p()
            if h is None:
                self.error = self.error or RuntimeError(f"rank {q} could not allocate its mailbox")
                ptrs.append(0)
                continue
            rc = lib.linrec_ipc_open(h, C.byref(p))
            if rc != capi.OK:
                self.error = self.error or capi.LinrecError(rc, lib.linrec_last_error().decode())
                ptrs.append(0)
                continue
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=device)  # device array of mailbox pointers
        self.epoch = [0, 0]

    def exchange(self, direction, consumers, sources, zero_a=False):
        """linrec_exchange_t of this step (epoch[direction] already advanced):
        consumers = (first, last) ranks receiving this rank's aggregate,
        sources = (first, last, step) ranks folded into the incoming carry."""
        return capi.Exchange(self.ptrs.data_ptr(), self.world, self.rank, self.epoch[direction],
                             consumers[0], consumers[1], sources[0], sources[1], sources[2], int(zero_a))

    def publish(self, agg, direction, q0, q1, stream):
        capi.check(capi.lib.linrec_p2p_publish_f32(agg.data_ptr(), self.W, self.world, self.rank, direction,
                                                   self.epoch[direction], self.ptrs.data_ptr(), q0, q1, stream))

    def compose(self, direction, local, first, last, step, seed, out, stream):
        capi.check(capi.lib.linrec_p2p_compose_f32(self.W, self.world, self.rank, direction, self.epoch[direction],
                                                   self.ptrs.data_ptr(), local.data_ptr(), first, last, step,
                                                   None if seed is None else seed.data_ptr(), out.data_ptr(), stream))

    def close(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p in self.opened:
            capi.lib.linrec_ipc_close(p)
        self.opened = []
        dist.barrier(group=self.group)
        if self.own:
            capi.lib.linrec_ipc_free(self.own)
            self.own = None


def _same_node(group) -> bool:
    import socket
    names = [None] * dist.get_world_size(group)
    dist.all_gather_object(names, socket.gethostname(), group=group)
    return len(set(names)) == 1


class SequenceShardedScan:
    """h = scan(lam, x, h0) and its gradients with T split across the ranks
    of `group`; rank r holds rows segment_bounds(T, world, r) of every
    [T, ...] tensor (fp32, C-contiguous, W = prod of the trailing dims).

    forward(lam, x, h0, h)                      h0 used on rank 0 only
    backward(lam, h0, h, dh, dlam, dx, dh0)     dh0 written on rank 0 only
    """

    def __init__(self, T, W, group=None, ws=None, stream=None, backend=None, device=None, exchange="auto"):
        """exchange: "p2p" (peer-memory mailboxes, csrc/p2p.cu), "collective"
        (all-gather) or "auto" (p2p when every rank is on this node and the
        CUDA backend runs)."""
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.T, self.W = T, W
        self.Tl = segment_rows(T, self.world, self.rank)
        self.be = backend if backend is not None else CudaBackend(ws, stream)
        self.stream = stream
        dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                                 if backend is None else torch.device("cpu"))
        f = dict(dtype=torch.float32, device=dev)
        self.rows_f = self.be.tile_rows(self.Tl, W, False)
        self.rows_b = self.be.tile_rows(self.Tl, W, True)
        nf = self.be.prod_rows(self.Tl, W, False)
        nb = self.be.prod_rows(self.Tl, W, True)
        with self._on_stream():  # filled on the stream the steps run on (no cross-stream read)
            self.seg_prod_f = torch.empty(nf, W, **f)
            self.seg_prod_b = torch.empty(nb, W, **f)
            self.agg = torch.empty(2, W, **f)
            self.aggs = torch.empty(self.world, 2, W, **f)
            self.c_in = torch.zeros(W, **f)
            self.y_in = torch.zeros(W, **f)
            self.dh0_loc = torch.empty(W, **f)
            self.ones = torch.ones(W, **f)
            self.zeros = torch.zeros(W, **f)
        self.hprev = None
        use_p2p = exchange == "p2p" or (exchange == "auto" and backend is None and self.world > 1
                                        and _same_node(self.group))
        self.mb = None
        if use_p2p:
            # every rank must agree on the exchange: a rank whose IPC setup
            # fails makes all of them fall back to the all-gather ("auto" only)
            self.mb = PeerMailboxes(W, self.group, dev)
            err = self.mb.error
            if exchange == "auto":
                ok = torch.tensor([0.0 if err is not None else 1.0],
                                  device=dev if dist.get_backend(self.group) == "nccl" else "cpu")
                dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
                if ok.item() < 1.0:
                    self.mb.close()
                    self.mb = None
                    use_p2p = False
            elif err is not None:
                self.mb.close()
                raise err
        self.exchange = "p2p" if use_p2p else "collective"
        # kernels launched per step on this rank (for bench.py's gpu_launches)
        r, R = self.rank, self.world
        # fwd: scan + finalize (+ fix-up when virtually segmented) + compose/fix-up
        # for r > 0; bwd likewise + the dh0 compose on rank 0
        # (an estimate; bench.py counts the launches on the device): the rank
        # aggregate is folded in the scan kernel's tail at W <= 256, else by a
        # fold kernel
        fold = 0 if (W <= 256 and W % 4 == 0) else 1
        if use_p2p:  # per direction: scan (+publish), [fold + publish], compose + fix-up (+ dh0 fold on rank 0)
            self.launches_per_step = 2 * (2 + fold) + (1 if r == 0 else 0)
        else:  # per direction: scan, [fold], compose of the gathered aggregates, fix-up
            self.launches_per_step = ((2 + fold + (1 if r > 0 else 0))
                                      + (2 + fold + (1 if r < R - 1 else 0) + (1 if r == 0 else 0)))

    def _on_stream(self):
        if self.stream is not None and torch.cuda.is_available() and isinstance(self.stream, torch.cuda.Stream):
            return torch.cuda.stream(self.stream)
        return contextlib.nullcontext()

    # -- collectives -----------------------------------------------------------
    def _all_gather(self, local, out):
        """all_gather of a small [..] tensor into out[world, ..]: NCCL over
        NVLink on device buffers; gloo (CPU tests, or several ranks sharing
        one GPU in tests) through host copies."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(out.view(-1), local.reshape(-1), group=self.group)
            return
        if local.is_cuda:
            parts = [torch.empty_like(local, device="cpu") for _ in range(self.world)]
            dist.all_gather(parts, local.cpu(), group=self.group)
            out.copy_(torch.stack(parts).to(out.device))
        else:
            parts = list(out.unbind(0))
            dist.all_gather(parts, local, group=self.group)

    # -- forward -------------------------------------------------------------------
    def forward(self, lam, x, h0, h):
        """Rank r scans its segment; c_in (the true h before the segment) is
        kept for the backward (hprev)."""
        with self._on_stream():
            return self._forward(lam, x, h0, h)

    def _forward(self, lam, x, h0, h):
        r, R, W, T = self.rank, self.world, self.W, self.Tl
        if self.mb is not None:
            # the exchange runs inside the fold (publish) and the fix-up (compose)
            self.mb.epoch[0] += 1
            ex = self.mb.exchange(0, (r + 1, R), (0, r, 1), zero_a=(r == 0))
            self.be.segment_scan_exchange(lam, x, h0 if r == 0 else None, h, self.seg_prod_f, self.agg, T, W, ex)
            self.be.fixup_exchange(lam, h, self.seg_prod_f, self.c_in, T, W, self.rows_f, ex)
            self.hprev = self.c_in if r > 0 else (h0 if h0 is not None else self.zeros)
            return h
        self.be.segment_scan(lam, x, h0 if r == 0 else None, h, self.seg_prod_f, self.agg, T, W)
        if r == 0:
            self.agg[0].zero_()  # h0 is already folded into rank 0's segment
        self._all_gather(self.agg, self.aggs)
        if r > 0:
            self.be.compose(self.aggs, 0, r, 1, None, self.c_in, W)
        # always: the fix-up also stitches the segment's own virtual segments
        self.be.fixup(lam, h, self.seg_prod_f, self.c_in if r > 0 else None, T, W, self.rows_f)
        if r > 0:
            self.hprev = self.c_in
        else:
            self.hprev = h0 if h0 is not None else self.zeros
        return h

    # -- backward ------------------------------------------------------------------
    def backward(self, lam, h0, h, dh, dlam, dx, dh0, hprev=None):
        """Gradients of the sharded recurrence.  hprev (the true h row before
        the segment) defaults to the one the last forward() computed; pass it
        explicitly when calling backward alone."""
        with self._on_stream():
            return self._backward(lam, h0, h, dh, dlam, dx, dh0, hprev)

    def _backward(self, lam, h0, h, dh, dlam, dx, dh0, hprev):
        r, R, W, T = self.rank, self.world, self.W, self.Tl
        if hprev is None:
            hprev = self.hprev if self.hprev is not None else self._halo(h, h0)
        lam_next = self.ones if r < R - 1 else None
        if r == R - 1:
            self.y_in.zero_()
        if self.mb is not None:
            self.mb.epoch[1] += 1
            ex = self.mb.exchange(1, (0, r), (R - 1, r, -1))
            self.be.segment_scan_backward_exchange(lam, hprev, h, dh, lam_next, dlam, dx, self.dh0_loc,
                                                   self.seg_prod_b, self.agg, T, W, ex)
            self.be.fixup_backward_exchange(lam, hprev, h, lam_next, self.seg_prod_b, self.y_in, dlam, dx, T, W,
                                            self.rows_b, ex)
        else:
            self.be.segment_scan_backward(lam, hprev, h, dh, lam_next, dlam, dx, self.dh0_loc, self.seg_prod_b,
                                          self.agg, T, W)
            self._all_gather(self.agg, self.aggs)
            if r < R - 1:
                self.be.compose(self.aggs, R - 1, r, -1, None, self.y_in, W)
            self.be.fixup_backward(lam, hprev, h, lam_next, self.seg_prod_b, self.y_in if r < R - 1 else None,
                                   dlam, dx, T, W, self.rows_b)
        if r == 0 and dh0 is not None:
            # own aggregate only: the local fold of the all-gather path
            self.aggs[0].copy_(self.agg)
            self.be.compose(self.aggs, 0, 1, 1, self.y_in, dh0.view(-1), W)
        return dlam, dx, dh0

    def close(self):
        if self.mb is not None:
            self.mb.close()
            self.mb = None

    def _halo(self, h, h0):
        """True h row before this segment: last row of the previous rank's h."""
        rows = torch.empty(self.world, self.W, dtype=h.dtype, device=h.device)
        self._all_gather(h[-1].reshape(self.W).contiguous(), rows)
        if self.rank == 0:
            return h0.reshape(self.W) if h0 is not None else self.zeros
        return rows[self.rank - 1].clone()
