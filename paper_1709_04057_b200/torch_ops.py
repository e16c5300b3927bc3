"""torch CUDA tensors -> the sm_100a scans (C ABI), on torch's current stream.

torch is plumbing here (device memory, streams); every FLOP runs in
liblinrec_cuda.so.  Tensors must be CUDA, C-contiguous, float32/float64,
shaped [T, batch, features] (h0: [batch, features]).
"""
from __future__ import annotations

import torch

from . import capi


def _check(t, name, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.float32, torch.float64):
        raise TypeError("decays must be float32 or float64")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: all arrays must share the decays dtype")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous")


def _dims(lam):
    if lam.dim() != 3:
        raise ValueError("decays must have shape [T, batch, features]")
    T = lam.shape[0]
    W = lam.numel() // T if T else 0
    return T, W


def _check_like(t, name, shape):
    """Exact-shape check for h0 / out buffers: the C ABI only sees pointers
    and reads or writes T*W (or W) elements, so a mis-sized tensor must be
    rejected here with the reference's contract message
    (recurrence.hpp:39-51 validate_recurrence_shapes)."""
    if list(t.shape) != list(shape):
        if name == "initial":
            raise RuntimeError(f"recurrence: initial state {list(t.shape)} does not match {list(shape)}")
        raise RuntimeError(f"{name}: shape mismatch, {list(shape)} vs {list(t.shape)}")


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _screen(t, name):
    """check_finite (recurrence.hpp:133-163): RuntimeError naming the first
    non-finite element, "non-finite value in <name> at [t=.., b=.., n=..]"."""
    if t is None:
        return
    if t.dim() == 3:
        T, b, n = t.shape
    else:
        T, (b, n) = 0, t.shape
    try:
        capi.screen_finite(t.data_ptr(), T, b, n, name, t.element_size(), _stream())
    except capi.LinrecError as e:
        raise RuntimeError(str(e)) from None


def scan(lam, x, h0=None, mode="parallel", out=None, ws=None, check_finite=False):
    _check(lam, "decays")
    _check(x, "impulses", lam.dtype)
    if lam.shape != x.shape:
        raise RuntimeError(f"recurrence: shape mismatch, {list(lam.shape)} vs {list(x.shape)}")
    T, W = _dims(lam)
    if h0 is not None:
        _check(h0, "initial", lam.dtype)
        _check_like(h0, "initial", lam.shape[1:])
    if out is None:
        h = torch.empty_like(lam)
    else:
        h = out
        _check(h, "out", lam.dtype)
        _check_like(h, "out", lam.shape)
    if check_finite:  # screen_recurrence (recurrence.hpp:157-163)
        _screen(lam, "decays")
        _screen(x, "impulses")
        _screen(h0, "initial")
    capi.scan(lam.data_ptr(), x.data_ptr(), _ptr(h0), h.data_ptr(), T, W,
              capi.SERIAL if mode == "serial" else capi.PARALLEL, lam.element_size(),
              None if ws is None else ws.handle, _stream())
    return h


def scan_backward(lam, h0, h, dh, mode="parallel", out=None, ws=None, check_finite=False):
    _check(lam, "decays")
    for t, n in ((h, "h"), (dh, "d_h")):
        _check(t, n, lam.dtype)
        if t.shape != lam.shape:
            raise RuntimeError(f"scan_backward({n}): shape mismatch, {list(lam.shape)} vs {list(t.shape)}")
    T, W = _dims(lam)
    if h0 is not None:
        _check(h0, "initial", lam.dtype)
        _check_like(h0, "initial", lam.shape[1:])
    if out is None:
        dlam, dx = torch.empty_like(lam), torch.empty_like(lam)
        dh0 = torch.empty(lam.shape[1:], dtype=lam.dtype, device=lam.device)
    else:
        dlam, dx, dh0 = out
        for t, n, shp in ((dlam, "d_decays", lam.shape), (dx, "d_impulses", lam.shape),
                          (dh0, "d_initial", lam.shape[1:])):
            _check(t, n, lam.dtype)
            _check_like(t, n, shp)
    if check_finite:  # recurrence.hpp:292-296
        _screen(lam, "decays")
        _screen(dh, "d_h")
    capi.scan_backward(lam.data_ptr(), _ptr(h0), h.data_ptr(), dh.data_ptr(), dlam.data_ptr(),
                       dx.data_ptr(), dh0.data_ptr(), T, W,
                       capi.SERIAL if mode == "serial" else capi.PARALLEL, lam.element_size(),
                       None if ws is None else ws.handle, _stream())
    return dlam, dx, dh0


class LinearRecurrence(torch.autograd.Function):
    """Autograd wrapper: h = scan(lam, x, h0) with the fused reverse scan."""

    @staticmethod
    def forward(ctx, lam, x, h0):
        lam = lam.contiguous()
        h0 = None if h0 is None else h0.contiguous()
        h = scan(lam, x.contiguous(), h0)
        ctx.save_for_backward(lam, h, h0 if h0 is not None else torch.empty(0, device=lam.device))
        ctx.has_h0 = h0 is not None
        return h

    @staticmethod
    def backward(ctx, dh):
        lam, h, h0 = ctx.saved_tensors
        dlam, dx, dh0 = scan_backward(lam, h0 if ctx.has_h0 else None, h, dh.contiguous())
        return dlam, dx, (dh0 if ctx.has_h0 else None)


def linear_recurrence(lam, x, h0=None):
    return LinearRecurrence.apply(lam, x, h0)
