"""GILR and GILR-LSTM layers on the B200 (reference: proj/include/linrec/layers.hpp).

Same names and semantics as the reference's layer API, over torch CUDA
tensors on the current stream; every FLOP runs in liblinrec_cuda.so (the
tcgen05 gate GEMMs with fused activation epilogues and the chained scans):

    gilr_init / gilr_forward / gilr_backward                  layers.hpp:42-133
    gilr_lstm_init / gilr_lstm_forward / gilr_lstm_backward   layers.hpp:165-375
    qrnn_init / qrnn_forward / qrnn_backward                  layers.hpp:376-548

Parameters are row-major exactly as GilrParams / GilrLstmParams (gate blocks
f, i, o, z stacked along the rows of U, V, bias).  Gradients ACCUMULATE into
the grads objects (tensor.hpp:272-296); dx is returned.  ``precision`` is
"fp32" (3xTF32 on the tensor cores, fp32-grade; default) or "tf32" (one TF32
pass, ~1e-3 relative).  Inputs: x [T, b, m] fp32 contiguous, or fp64: then
every parameter, state and adjoint is fp64 too and the call runs the
double-precision entry points (linrec_*_f64: fp64 CUDA-core GEMMs and the
fp64 scans; ``precision`` does not apply) -- the reference's layers are
templated on S and its test_layers.cpp runs them in double.  Widths that
are not multiples of 4 (the kernels' 16-byte TMA rows) are zero-padded here:
padded input columns meet zero weights and padded hidden units start at 0,
see only zero weights and so stay exactly 0 -- outputs and gradients are the
unpadded problem's (``_Pad``).  ``GilrLstm`` wraps the pair as a
torch.nn.Module with autograd.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import capi

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
ACT = {"tanh": 0, "identity": 1, "relu": 2}
PRECISION = {"fp32": capi.PREC_FP32, "tf32": capi.PREC_TF32}
MODE = {"serial": capi.SERIAL, "parallel": capi.PARALLEL}


class _GilrParamsC(C.Structure):
    _fields_ = [("U", _vp), ("V", _vp), ("b_g", _vp), ("b_z", _vp), ("act", _int)]


class _GilrGradsC(C.Structure):
    _fields_ = [("U", _vp), ("V", _vp), ("b_g", _vp), ("b_z", _vp)]


class _LstmParamsC(C.Structure):
    _fields_ = [("surrogate", _GilrParamsC), ("U", _vp), ("V", _vp), ("bias", _vp)]


class _LstmGradsC(C.Structure):
    _fields_ = [("surrogate", _GilrGradsC), ("U", _vp), ("V", _vp), ("bias", _vp)]


class _LstmCacheC(C.Structure):
    _fields_ = [("sg", _vp), ("si", _vp), ("htil", _vp), ("gates", _vp), ("c", _vp)]


def _bind():
    lib = capi.lib
    if getattr(lib, "_layers_bound", False):
        return lib
    lib.linrec_gilr_scratch_bytes.restype = C.c_size_t
    lib.linrec_gilr_scratch_bytes.argtypes = [_i64] * 4
    lib.linrec_gilr_lstm_scratch_bytes.restype = C.c_size_t
    lib.linrec_gilr_lstm_scratch_bytes.argtypes = [_i64] * 4
    tail = [_i64] * 4 + [_int, _int, _vp, C.c_size_t, _vp]
    lib.linrec_gilr_forward_f32.argtypes = [C.POINTER(_GilrParamsC)] + [_vp] * 5 + tail
    lib.linrec_gilr_backward_f32.argtypes = ([C.POINTER(_GilrParamsC)] + [_vp] * 6 + [C.POINTER(_GilrGradsC)]
                                             + [_vp] * 2 + tail)
    lib.linrec_gilr_lstm_forward_f32.argtypes = ([C.POINTER(_LstmParamsC)] + [_vp] * 4 + [C.POINTER(_LstmCacheC)]
                                                 + tail)
    lib.linrec_gilr_lstm_backward_f32.argtypes = ([C.POINTER(_LstmParamsC)] + [_vp] * 3 + [C.POINTER(_LstmCacheC)]
                                                  + [_vp] + [C.POINTER(_LstmGradsC)] + [_vp] * 3 + tail)
    lib.linrec_profile_end.argtypes = [C.c_char_p, C.c_size_t]
    lib.linrec_qrnn_scratch_bytes.restype = C.c_size_t
    lib.linrec_qrnn_scratch_bytes.argtypes = [_i64] * 5
    qtail = [_i64] * 5 + [_int, _int, _vp, C.c_size_t, _vp]
    lib.linrec_qrnn_forward_f32.argtypes = [_vp] * 7 + qtail
    lib.linrec_qrnn_backward_f32.argtypes = [_vp] * 10 + qtail
    # fp64 entry points: the same structs (void* fields), no precision argument
    for nm in ("linrec_gilr_scratch_bytes_f64", "linrec_gilr_lstm_scratch_bytes_f64"):
        getattr(lib, nm).restype = C.c_size_t
        getattr(lib, nm).argtypes = [_i64] * 4
    lib.linrec_qrnn_scratch_bytes_f64.restype = C.c_size_t
    lib.linrec_qrnn_scratch_bytes_f64.argtypes = [_i64] * 5
    tail64 = [_i64] * 4 + [_int, _vp, C.c_size_t, _vp]
    lib.linrec_gilr_forward_f64.argtypes = [C.POINTER(_GilrParamsC)] + [_vp] * 5 + tail64
    lib.linrec_gilr_backward_f64.argtypes = ([C.POINTER(_GilrParamsC)] + [_vp] * 6 + [C.POINTER(_GilrGradsC)]
                                             + [_vp] * 2 + tail64)
    lib.linrec_gilr_lstm_forward_f64.argtypes = ([C.POINTER(_LstmParamsC)] + [_vp] * 4 + [C.POINTER(_LstmCacheC)]
                                                 + tail64)
    lib.linrec_gilr_lstm_backward_f64.argtypes = ([C.POINTER(_LstmParamsC)] + [_vp] * 3 + [C.POINTER(_LstmCacheC)]
                                                  + [_vp] + [C.POINTER(_LstmGradsC)] + [_vp] * 3 + tail64)
    qtail64 = [_i64] * 5 + [_int, _vp, C.c_size_t, _vp]
    lib.linrec_qrnn_forward_f64.argtypes = [_vp] * 7 + qtail64
    lib.linrec_qrnn_backward_f64.argtypes = [_vp] * 10 + qtail64
    lib.linrec_gemm_f64.argtypes = [_vp, _int, _i64, _vp, _int, _i64, _vp, _i64, _i64, _i64, _i64, _int, _vp]
    lib._layers_bound = True
    return lib


def profile_begin():
    """Start per-stage timing of the layer calls on this thread (CUDA events
    on each call's stream)."""
    capi.check(_bind().linrec_profile_begin())


def profile_end() -> dict:
    """Stop timing; returns {stage: (total_ms, count)} in first-seen order."""
    buf = C.create_string_buffer(1 << 16)
    capi.check(_bind().linrec_profile_end(buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        name, ms, cnt = line.split()
        out[name] = (float(ms), int(cnt))
    return out


def _p(t):
    return None if t is None else t.data_ptr()


def _check_f32(t, name, dtype=None):
    """CUDA, C-contiguous, and float32 -- or `dtype` (the call's dtype, taken
    from x: float32 or float64, no silent cast, linrec_py.cpp:21-29)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    want = torch.float32 if dtype is None else dtype
    if want not in (torch.float32, torch.float64):
        raise TypeError(f"{name}: the layers run float32 or float64, got {want}")
    if t.dtype != want:
        raise TypeError(f"{name} must be {str(want).replace('torch.', '')} like x")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be C-contiguous")


def _check_shape(t, name, shape, dtype=None):
    """The C ABI sees raw pointers only: an initial state, adjoint or cache
    of the wrong shape would be an out-of-bounds device access, so reject it
    with the reference's contract error (layers.hpp check_same_shape /
    tensor.hpp:168-189)."""
    if t is None:
        return
    _check_f32(t, name, dtype)
    if list(t.shape) != list(shape):
        raise RuntimeError(f"{name}: shape mismatch, {list(shape)} vs {list(t.shape)}")


_scratch = {}


def _scratch_for(nbytes, device):
    """Per-(device, stream) scratch, grown on demand (torch caching allocator)."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _scratch.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
        _scratch[key] = buf
    return buf


def release_scratch():
    _scratch.clear()


# ---- parameters (layers.hpp:30-76, :146-211) ---------------------------------
@dataclass
class GilrParams:
    U: torch.Tensor    # [n, m]
    V: torch.Tensor    # [n, m]
    b_g: torch.Tensor  # [n]
    b_z: torch.Tensor  # [n]
    act: str = "tanh"

    def input(self):
        return self.U.shape[1]

    def hidden(self):
        return self.U.shape[0]

    def tensors(self):
        return [self.U, self.V, self.b_g, self.b_z]

    def _c(self):
        return _GilrParamsC(_p(self.U), _p(self.V), _p(self.b_g), _p(self.b_z), ACT[self.act])


@dataclass
class GilrGrads:
    U: torch.Tensor
    V: torch.Tensor
    b_g: torch.Tensor
    b_z: torch.Tensor

    @staticmethod
    def zeros_like(p: GilrParams) -> "GilrGrads":
        return GilrGrads(*(torch.zeros_like(t) for t in p.tensors()))

    def tensors(self):
        return [self.U, self.V, self.b_g, self.b_z]

    def _c(self):
        return _GilrGradsC(_p(self.U), _p(self.V), _p(self.b_g), _p(self.b_z))


@dataclass
class GilrLstmParams:
    surrogate: GilrParams
    U: torch.Tensor     # [4n, n]
    V: torch.Tensor     # [4n, m]
    bias: torch.Tensor  # [4n]

    def input(self):
        return self.V.shape[1]

    def hidden(self):
        return self.U.shape[1]

    def tensors(self):
        return self.surrogate.tensors() + [self.U, self.V, self.bias]

    def _c(self):
        return _LstmParamsC(self.surrogate._c(), _p(self.U), _p(self.V), _p(self.bias))


@dataclass
class GilrLstmGrads:
    surrogate: GilrGrads
    U: torch.Tensor
    V: torch.Tensor
    bias: torch.Tensor

    @staticmethod
    def zeros_like(p: GilrLstmParams) -> "GilrLstmGrads":
        return GilrLstmGrads(GilrGrads.zeros_like(p.surrogate), torch.zeros_like(p.U), torch.zeros_like(p.V),
                             torch.zeros_like(p.bias))

    def tensors(self):
        return self.surrogate.tensors() + [self.U, self.V, self.bias]

    def _c(self):
        return _LstmGradsC(self.surrogate._c(), _p(self.U), _p(self.V), _p(self.bias))


@dataclass
class GilrCache:
    g: torch.Tensor = None
    i: torch.Tensor = None
    h: torch.Tensor = None


@dataclass
class GilrLstmCache:
    """GilrLstmCache (layers.hpp:183-188) on the device.  htil is [T+1, b, n]
    (row 0 = htil0) so htil_prev = htil[:-1] without a copy; gates are the
    four activated planes [4, T, b, n] (the reference interleaves them as
    [T, b, 4n]; ``gates_interleaved()`` gives that view)."""
    sg: torch.Tensor = None
    si: torch.Tensor = None
    htil: torch.Tensor = None
    gates: torch.Tensor = None
    c: torch.Tensor = None

    def allocate(self, T, b, n, device, dtype=torch.float32):
        if (self.c is not None and tuple(self.c.shape) == (T, b, n) and self.c.device == torch.device(device)
                and self.c.dtype == dtype):
            return self  # reuse (e.g. one cache per layer across training steps)
        kw = dict(dtype=dtype, device=device)
        self.sg = torch.empty(T, b, n, **kw)
        self.si = torch.empty(T, b, n, **kw)
        self.htil = torch.empty(T + 1, b, n, **kw)
        self.gates = torch.empty(4, T, b, n, **kw)
        self.c = torch.empty(T, b, n, **kw)
        return self

    def check(self, T, b, n, dtype=None):
        """Shapes a backward pass reads through raw pointers."""
        for t, nm, shp in ((self.sg, "cache.sg", (T, b, n)), (self.si, "cache.si", (T, b, n)),
                           (self.htil, "cache.htil", (T + 1, b, n)), (self.gates, "cache.gates", (4, T, b, n)),
                           (self.c, "cache.c", (T, b, n))):
            if t is None:
                raise RuntimeError(f"{nm}: cache not filled by a forward pass")
            _check_shape(t, nm, shp, dtype)

    def surrogate_h(self):
        return self.htil[1:]

    def htil_prev(self):
        return self.htil[:-1]

    def gates_interleaved(self):
        return self.gates.permute(1, 2, 0, 3).reshape(self.gates.shape[1], self.gates.shape[2], -1)

    def _c(self):
        return _LstmCacheC(_p(self.sg), _p(self.si), _p(self.htil), _p(self.gates), _p(self.c))


def _uniform(gen, rows, cols, scale, device, dtype=torch.float32):
    return ((torch.rand(rows, cols, generator=gen, dtype=torch.float64) * 2 - 1) * scale).to(
        device=device, dtype=dtype)


def gilr_init(gen: torch.Generator, m: int, n: int, gate_bias: float = 1.0, device="cuda",
              act: str = "tanh", dtype=torch.float32) -> GilrParams:
    """gilr_init (layers.hpp:42-55): U, V ~ U(+-1/sqrt(m)), b_g = gate_bias, b_z = 0."""
    s = 1.0 / math.sqrt(m)
    return GilrParams(_uniform(gen, n, m, s, device, dtype), _uniform(gen, n, m, s, device, dtype),
                      torch.full((n,), gate_bias, dtype=dtype, device=device),
                      torch.zeros(n, dtype=dtype, device=device), act)


def gilr_lstm_init(gen: torch.Generator, m: int, n: int, gate_bias: float = 1.0, device="cuda",
                   dtype=torch.float32) -> GilrLstmParams:
    """gilr_lstm_init (layers.hpp:165-176): surrogate as gilr_init, U ~ U(+-1/sqrt(n)),
    V ~ U(+-1/sqrt(m)), bias = gate_bias on the f block."""
    sur = gilr_init(gen, m, n, gate_bias, device, dtype=dtype)
    bias = torch.zeros(4 * n, dtype=dtype, device=device)
    bias[:n] = gate_bias
    return GilrLstmParams(sur, _uniform(gen, 4 * n, n, 1.0 / math.sqrt(n), device, dtype),
                          _uniform(gen, 4 * n, m, 1.0 / math.sqrt(m), device, dtype), bias)


def _f64(x) -> bool:
    return isinstance(x, torch.Tensor) and x.dtype == torch.float64


def _dims(x, n):
    _check_f32(x, "x", x.dtype if _f64(x) else None)
    if x.dim() != 3:
        raise ValueError("x must have shape [T, batch, features]")
    T, b, m = x.shape
    return T, b, m, n


def _call(rc):
    capi.check(rc)


# ---- GILR ------------------------------------------------------------------------
def _gilr_forward_core(p: GilrParams, x, h0=None, mode="parallel", precision="fp32", cache: GilrCache | None = None):
    """gilr_forward (layers.hpp:78-100) -> h [T, b, n]; fills ``cache`` (g, i, h)."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    if m != p.input():
        raise RuntimeError("gilr_forward: input feature mismatch")
    dt = x.dtype
    for t, nm in zip(p.tensors(), ("U", "V", "b_g", "b_z")):
        _check_f32(t, nm, dt)
    _check_shape(h0, "h0", (b, n), dt)
    dev = x.device
    h = torch.empty(T, b, n, dtype=dt, device=dev)
    g = torch.empty_like(h)
    i = torch.empty_like(h)
    pc = p._c()
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_gilr_scratch_bytes_f64(T, b, m, n), dev)
        _call(lib.linrec_gilr_forward_f64(C.byref(pc), _p(x), _p(h0), _p(h), _p(g), _p(i), T, b, m, n, MODE[mode],
                                          _p(scr), scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_gilr_scratch_bytes(T, b, m, n), dev)
        _call(lib.linrec_gilr_forward_f32(C.byref(pc), _p(x), _p(h0), _p(h), _p(g), _p(i), T, b, m, n, MODE[mode],
                                          PRECISION[precision], _p(scr), scr.numel(), st))
    if cache is not None:
        cache.g, cache.i, cache.h = g, i, h
    return h


def _gilr_backward_core(p: GilrParams, x, h0, cache: GilrCache, d_h, grads: GilrGrads, mode="parallel",
                  precision="fp32", want_dh0=True):
    """gilr_backward (layers.hpp:102-133): accumulates into ``grads``; returns (dx, dh0)."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    dt = x.dtype
    _check_shape(d_h, "d_h", (T, b, n), dt)
    _check_shape(h0, "h0", (b, n), dt)
    for t, nm in ((cache.g, "cache.g"), (cache.i, "cache.i"), (cache.h, "cache.h")):
        _check_shape(t, nm, (T, b, n), dt)
    for t, nm in zip(p.tensors() + grads.tensors(), ("U", "V", "b_g", "b_z") * 2):
        if t is not None:
            _check_f32(t, nm, dt)
    dev = x.device
    dx = torch.empty(T, b, m, dtype=dt, device=dev)
    dh0 = torch.empty(b, n, dtype=dt, device=dev) if want_dh0 else None
    pc, gc = p._c(), grads._c()
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_gilr_scratch_bytes_f64(T, b, m, n), dev)
        _call(lib.linrec_gilr_backward_f64(C.byref(pc), _p(x), _p(h0), _p(cache.g), _p(cache.i), _p(cache.h),
                                           _p(d_h), C.byref(gc), _p(dx), _p(dh0), T, b, m, n, MODE[mode], _p(scr),
                                           scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_gilr_scratch_bytes(T, b, m, n), dev)
        _call(lib.linrec_gilr_backward_f32(C.byref(pc), _p(x), _p(h0), _p(cache.g), _p(cache.i), _p(cache.h),
                                           _p(d_h), C.byref(gc), _p(dx), _p(dh0), T, b, m, n, MODE[mode],
                                           PRECISION[precision], _p(scr), scr.numel(), st))
    return dx, dh0


# ---- GILR-LSTM ---------------------------------------------------------------------
def _gilr_lstm_forward_core(p: GilrLstmParams, x, htil0=None, c0=None, mode="parallel", precision="fp32",
                      cache: GilrLstmCache | None = None):
    """gilr_lstm_forward (layers.hpp:245-293) -> h [T, b, n]; fills ``cache``."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    if m != p.input():
        raise RuntimeError("gilr_lstm_forward: input feature mismatch")
    dt = x.dtype
    for t in p.tensors():
        _check_f32(t, "parameter", dt)
    for t, nm in ((htil0, "htil0"), (c0, "c0")):
        _check_shape(t, nm, (b, n), dt)
    dev = x.device
    if cache is None:
        cache = GilrLstmCache()
    cache.allocate(T, b, n, dev, dt)
    h = torch.empty(T, b, n, dtype=dt, device=dev)
    pc, cc = p._c(), cache._c()
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_gilr_lstm_scratch_bytes_f64(T, b, m, n), dev)
        _call(lib.linrec_gilr_lstm_forward_f64(C.byref(pc), _p(x), _p(htil0), _p(c0), _p(h), C.byref(cc), T, b, m,
                                               n, MODE[mode], _p(scr), scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_gilr_lstm_scratch_bytes(T, b, m, n), dev)
        _call(lib.linrec_gilr_lstm_forward_f32(C.byref(pc), _p(x), _p(htil0), _p(c0), _p(h), C.byref(cc), T, b, m,
                                               n, MODE[mode], PRECISION[precision], _p(scr), scr.numel(), st))
    return h


def _gilr_lstm_backward_core(p: GilrLstmParams, x, htil0, c0, cache: GilrLstmCache, d_h, grads: GilrLstmGrads,
                       mode="parallel", precision="fp32", want_initial=True):
    """gilr_lstm_backward (layers.hpp:295-375): accumulates into ``grads``;
    returns (dx, d_htil0, d_c0)."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    dt = x.dtype
    _check_shape(d_h, "d_h", (T, b, n), dt)
    for t, nm in ((htil0, "htil0"), (c0, "c0")):
        _check_shape(t, nm, (b, n), dt)
    cache.check(T, b, n, dt)
    for t in p.tensors() + grads.tensors():
        if t is not None:
            _check_f32(t, "parameter", dt)
    dev = x.device
    dx = torch.empty(T, b, m, dtype=dt, device=dev)
    dht0 = torch.empty(b, n, dtype=dt, device=dev) if want_initial else None
    dc0 = torch.empty(b, n, dtype=dt, device=dev) if want_initial else None
    pc, cc, gc = p._c(), cache._c(), grads._c()
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_gilr_lstm_scratch_bytes_f64(T, b, m, n), dev)
        _call(lib.linrec_gilr_lstm_backward_f64(C.byref(pc), _p(x), _p(htil0), _p(c0), C.byref(cc), _p(d_h),
                                                C.byref(gc), _p(dx), _p(dht0), _p(dc0), T, b, m, n, MODE[mode],
                                                _p(scr), scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_gilr_lstm_scratch_bytes(T, b, m, n), dev)
        _call(lib.linrec_gilr_lstm_backward_f32(C.byref(pc), _p(x), _p(htil0), _p(c0), C.byref(cc), _p(d_h),
                                                C.byref(gc), _p(dx), _p(dht0), _p(dc0), T, b, m, n, MODE[mode],
                                                PRECISION[precision], _p(scr), scr.numel(), st))
    return dx, dht0, dc0


# ---- QRNN (layers.hpp:376-548) -----------------------------------------------------------
@dataclass
class QrnnParams:
    """QrnnParams (layers.hpp:390-405): k taps W_s [3n, m] (blocks f, o, z),
    stored packed as W [k, 3n, m] (W[s] sees x_{t-s}); bias [3n]."""
    W: torch.Tensor
    bias: torch.Tensor

    def input(self):
        return self.W.shape[2]

    def hidden(self):
        return self.bias.shape[0] // 3

    def window(self):
        return self.W.shape[0]

    def tensors(self):
        return [self.W, self.bias]


@dataclass
class QrnnGrads:
    W: torch.Tensor
    bias: torch.Tensor

    @staticmethod
    def zeros_like(p: QrnnParams) -> "QrnnGrads":
        return QrnnGrads(torch.zeros_like(p.W), torch.zeros_like(p.bias))

    def tensors(self):
        return [self.W, self.bias]


@dataclass
class QrnnCache:
    """QrnnCache (layers.hpp:420-423): gates [3, T, b, n] activated f, o, z
    planes (the reference interleaves them as [T, b, 3n]), c [T, b, n]."""
    gates: torch.Tensor = None
    c: torch.Tensor = None

    def gates_interleaved(self):
        return self.gates.permute(1, 2, 0, 3).reshape(self.gates.shape[1], self.gates.shape[2], -1)


def qrnn_init(gen: torch.Generator, m: int, n: int, k: int, gate_bias: float = 1.0, device="cuda",
              dtype=torch.float32) -> QrnnParams:
    """qrnn_init (layers.hpp:411-422): W_s ~ U(+-1/sqrt(m k)), bias = gate_bias on f."""
    if k < 1:
        raise RuntimeError("qrnn_init: window must be >= 1")
    s = 1.0 / math.sqrt(m * k)
    W = torch.stack([_uniform(gen, 3 * n, m, s, device, dtype) for _ in range(k)])
    bias = torch.zeros(3 * n, dtype=dtype, device=device)
    bias[:n] = gate_bias
    return QrnnParams(W.contiguous(), bias)


def _qrnn_forward_core(p: QrnnParams, x, c0=None, mode="parallel", precision="fp32", cache: QrnnCache | None = None):
    """qrnn_forward (layers.hpp:449-494) -> h [T, b, n]; fills ``cache``."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    k = p.window()
    if m != p.input():
        raise RuntimeError("qrnn_forward: input feature mismatch")
    if k > T:
        raise RuntimeError("qrnn_forward: filter window exceeds sequence length")
    dt = x.dtype
    for t, nm in ((p.W, "W"), (p.bias, "bias")):
        _check_f32(t, nm, dt)
    _check_shape(c0, "c0", (b, n), dt)
    dev = x.device
    if cache is None:
        cache = QrnnCache()
    if cache.c is None or tuple(cache.c.shape) != (T, b, n) or cache.c.dtype != dt:
        cache.gates = torch.empty(3, T, b, n, dtype=dt, device=dev)
        cache.c = torch.empty(T, b, n, dtype=dt, device=dev)
    h = torch.empty(T, b, n, dtype=dt, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_qrnn_scratch_bytes_f64(T, b, m, n, k), dev)
        _call(lib.linrec_qrnn_forward_f64(_p(p.W), _p(p.bias), _p(x), _p(c0), _p(h), _p(cache.gates), _p(cache.c),
                                          T, b, m, n, k, MODE[mode], _p(scr), scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_qrnn_scratch_bytes(T, b, m, n, k), dev)
        _call(lib.linrec_qrnn_forward_f32(_p(p.W), _p(p.bias), _p(x), _p(c0), _p(h), _p(cache.gates), _p(cache.c),
                                          T, b, m, n, k, MODE[mode], PRECISION[precision], _p(scr), scr.numel(), st))
    return h


def _qrnn_backward_core(p: QrnnParams, x, c0, cache: QrnnCache, d_h, grads: QrnnGrads, mode="parallel",
                  precision="fp32", want_dc0=True):
    """qrnn_backward (layers.hpp:496-548): accumulates into ``grads``; returns (dx, dc0)."""
    lib = _bind()
    T, b, m, n = _dims(x, p.hidden())
    k = p.window()
    dt = x.dtype
    _check_shape(d_h, "d_h", (T, b, n), dt)
    _check_shape(c0, "c0", (b, n), dt)
    _check_shape(cache.gates, "cache.gates", (3, T, b, n), dt)
    _check_shape(cache.c, "cache.c", (T, b, n), dt)
    for t, nm in ((p.W, "W"), (grads.W, "grads.W"), (grads.bias, "grads.bias")):
        if t is not None:
            _check_f32(t, nm, dt)
    dev = x.device
    dx = torch.empty(T, b, m, dtype=dt, device=dev)
    dc0 = torch.empty(b, n, dtype=dt, device=dev) if want_dc0 else None
    st = torch.cuda.current_stream(dev).cuda_stream
    if _f64(x):
        scr = _scratch_for(lib.linrec_qrnn_scratch_bytes_f64(T, b, m, n, k), dev)
        _call(lib.linrec_qrnn_backward_f64(_p(p.W), _p(x), _p(c0), _p(cache.gates), _p(cache.c), _p(d_h),
                                           _p(grads.W), _p(grads.bias), _p(dx), _p(dc0), T, b, m, n, k, MODE[mode],
                                           _p(scr), scr.numel(), st))
    else:
        scr = _scratch_for(lib.linrec_qrnn_scratch_bytes(T, b, m, n, k), dev)
        _call(lib.linrec_qrnn_backward_f32(_p(p.W), _p(x), _p(c0), _p(cache.gates), _p(cache.c), _p(d_h),
                                           _p(grads.W), _p(grads.bias), _p(dx), _p(dc0), T, b, m, n, k, MODE[mode],
                                           PRECISION[precision], _p(scr), scr.numel(), st))
    return dx, dc0


# ---- torch autograd / nn.Module ---------------------------------------------------------
class _GilrLstmFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, htil0, c0, sU, sV, sbg, sbz, U, V, bias, precision):
        p = GilrLstmParams(GilrParams(sU, sV, sbg, sbz), U, V, bias)
        cache = GilrLstmCache()
        h = gilr_lstm_forward(p, x.contiguous(), htil0, c0, precision=precision, cache=cache)
        ctx.p, ctx.cache, ctx.precision = p, cache, precision
        ctx.save_for_backward(x, htil0, c0)
        return h

    @staticmethod
    def backward(ctx, dh):
        x, htil0, c0 = ctx.saved_tensors
        p = ctx.p
        grads = GilrLstmGrads.zeros_like(p)
        dx, dht0, dc0 = gilr_lstm_backward(p, x, htil0, c0, ctx.cache, dh.contiguous(), grads,
                                           precision=ctx.precision)
        return (dx, dht0, dc0, *grads.tensors(), None)


class GilrLstm(torch.nn.Module):
    """One GILR-LSTM layer (m -> n) with B200 forward/backward."""

    def __init__(self, m, n, gate_bias=1.0, seed=0, device="cuda", precision="fp32"):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        p = gilr_lstm_init(gen, m, n, gate_bias, device)
        self.names = ["sU", "sV", "sbg", "sbz", "U", "V", "bias"]
        for nm, t in zip(self.names, p.tensors()):
            self.register_parameter(nm, torch.nn.Parameter(t))
        self.precision = precision
        self.n = n

    def forward(self, x, htil0=None, c0=None):
        T, b, _ = x.shape
        z = torch.zeros(b, self.n, device=x.device, dtype=x.dtype)
        htil0 = z if htil0 is None else htil0
        c0 = z if c0 is None else c0
        return _GilrLstmFn.apply(x, htil0, c0, *[getattr(self, nm) for nm in self.names], self.precision)


# ---- widths that are not multiples of 4 --------------------------------------------
def _r4(v: int) -> int:
    return (v + 3) // 4 * 4


class _Pad:
    """Zero padding of a layer problem to widths m4, n4 (multiples of 4).
    Gate blocks stacked along rows (f, i, o, z / f, o, z, per tap) are padded
    block by block, so every block keeps its place."""

    def __init__(self, m, n):
        self.m, self.n, self.m4, self.n4 = m, n, _r4(m), _r4(n)

    def needed(self, x=None):
        if _f64(x):  # the fp64 entry points take any width
            return False
        return self.m4 != self.m or self.n4 != self.n

    def rows(self, t, blocks, cols, cols4):  # [blocks*n, cols] -> [blocks*n4, cols4]
        out = t.new_zeros(blocks, self.n4, cols4)
        out[:, :self.n, :cols] = t.reshape(blocks, self.n, cols)
        return out.reshape(blocks * self.n4, cols4)

    def vec(self, t, blocks):  # [blocks*n] -> [blocks*n4]
        out = t.new_zeros(blocks, self.n4)
        out[:, :self.n] = t.reshape(blocks, self.n)
        return out.reshape(-1)

    def last(self, t, width, width4):  # zero-pad the last dimension
        if t is None:
            return None
        out = t.new_zeros(*t.shape[:-1], width4)
        out[..., :width] = t
        return out

    def add_rows(self, dst, src, blocks, cols, cols4):
        dst += src.reshape(blocks, self.n4, cols4)[:, :self.n, :cols].reshape(dst.shape)

    def add_vec(self, dst, src, blocks):
        dst += src.reshape(blocks, self.n4)[:, :self.n].reshape(dst.shape)

    # parameters
    def gilr(self, p: GilrParams) -> GilrParams:
        return GilrParams(self.rows(p.U, 1, self.m, self.m4), self.rows(p.V, 1, self.m, self.m4),
                          self.vec(p.b_g, 1), self.vec(p.b_z, 1), p.act)

    def lstm(self, p: GilrLstmParams) -> GilrLstmParams:
        return GilrLstmParams(self.gilr(p.surrogate), self.rows(p.U, 4, self.n, self.n4),
                              self.rows(p.V, 4, self.m, self.m4), self.vec(p.bias, 4))

    def qrnn(self, p: QrnnParams) -> QrnnParams:
        k = p.window()
        W = self.rows(p.W.reshape(3 * k * self.n, self.m), 3 * k, self.m, self.m4).reshape(k, 3 * self.n4, self.m4)
        return QrnnParams(W.contiguous(), self.vec(p.bias, 3))


def gilr_forward(p: GilrParams, x, h0=None, mode="parallel", precision="fp32", cache: GilrCache | None = None):
    """gilr_forward (layers.hpp:78-100) -> h [T, b, n]; fills ``cache`` (g, i, h)."""
    pad = _Pad(x.shape[-1] if x.dim() == 3 else p.input(), p.hidden())
    if not pad.needed(x):
        return _gilr_forward_core(p, x, h0, mode, precision, cache)
    if x.shape[-1] != p.input():
        raise RuntimeError("gilr_forward: input feature mismatch")
    inner = cache if cache is not None else GilrCache()
    h = _gilr_forward_core(pad.gilr(p), pad.last(x, pad.m, pad.m4), pad.last(h0, pad.n, pad.n4), mode, precision,
                           inner)
    return h[..., :pad.n].contiguous()


def gilr_backward(p: GilrParams, x, h0, cache: GilrCache, d_h, grads: GilrGrads, mode="parallel",
                  precision="fp32", want_dh0=True):
    """gilr_backward (layers.hpp:102-133): accumulates into ``grads``; returns (dx, dh0)."""
    pad = _Pad(p.input(), p.hidden())
    if not pad.needed(x):
        return _gilr_backward_core(p, x, h0, cache, d_h, grads, mode, precision, want_dh0)
    pp = pad.gilr(p)
    g4 = GilrGrads.zeros_like(pp)
    dx, dh0 = _gilr_backward_core(pp, pad.last(x, pad.m, pad.m4), pad.last(h0, pad.n, pad.n4), cache,
                                  pad.last(d_h, pad.n, pad.n4), g4, mode, precision, want_dh0)
    pad.add_rows(grads.U, g4.U, 1, pad.m, pad.m4)
    pad.add_rows(grads.V, g4.V, 1, pad.m, pad.m4)
    pad.add_vec(grads.b_g, g4.b_g, 1)
    pad.add_vec(grads.b_z, g4.b_z, 1)
    return dx[..., :pad.m].contiguous(), None if dh0 is None else dh0[..., :pad.n].contiguous()


def gilr_lstm_forward(p: GilrLstmParams, x, htil0=None, c0=None, mode="parallel", precision="fp32",
                      cache: GilrLstmCache | None = None):
    """gilr_lstm_forward (layers.hpp:245-293) -> h [T, b, n]; fills ``cache``
    (padded to the kernels' widths when m or n is not a multiple of 4)."""
    pad = _Pad(x.shape[-1] if x.dim() == 3 else p.input(), p.hidden())
    if not pad.needed(x):
        return _gilr_lstm_forward_core(p, x, htil0, c0, mode, precision, cache)
    if x.shape[-1] != p.input():
        raise RuntimeError("gilr_lstm_forward: input feature mismatch")
    h = _gilr_lstm_forward_core(pad.lstm(p), pad.last(x, pad.m, pad.m4), pad.last(htil0, pad.n, pad.n4),
                                pad.last(c0, pad.n, pad.n4), mode, precision,
                                cache if cache is not None else GilrLstmCache())
    return h[..., :pad.n].contiguous()


def gilr_lstm_backward(p: GilrLstmParams, x, htil0, c0, cache: GilrLstmCache, d_h, grads: GilrLstmGrads,
                       mode="parallel", precision="fp32", want_initial=True):
    """gilr_lstm_backward (layers.hpp:295-375): accumulates into ``grads``;
    returns (dx, d_htil0, d_c0)."""
    pad = _Pad(p.input(), p.hidden())
    if not pad.needed(x):
        return _gilr_lstm_backward_core(p, x, htil0, c0, cache, d_h, grads, mode, precision, want_initial)
    pp = pad.lstm(p)
    g4 = GilrLstmGrads.zeros_like(pp)
    dx, dht0, dc0 = _gilr_lstm_backward_core(pp, pad.last(x, pad.m, pad.m4), pad.last(htil0, pad.n, pad.n4),
                                             pad.last(c0, pad.n, pad.n4), cache, pad.last(d_h, pad.n, pad.n4), g4,
                                             mode, precision, want_initial)
    s, s4 = grads.surrogate, g4.surrogate
    pad.add_rows(s.U, s4.U, 1, pad.m, pad.m4)
    pad.add_rows(s.V, s4.V, 1, pad.m, pad.m4)
    pad.add_vec(s.b_g, s4.b_g, 1)
    pad.add_vec(s.b_z, s4.b_z, 1)
    pad.add_rows(grads.U, g4.U, 4, pad.n, pad.n4)
    pad.add_rows(grads.V, g4.V, 4, pad.m, pad.m4)
    pad.add_vec(grads.bias, g4.bias, 4)
    cut = lambda t: None if t is None else t[..., :pad.n].contiguous()  # noqa: E731
    return dx[..., :pad.m].contiguous(), cut(dht0), cut(dc0)


def qrnn_forward(p: QrnnParams, x, c0=None, mode="parallel", precision="fp32", cache: QrnnCache | None = None):
    """qrnn_forward (layers.hpp:449-494) -> h [T, b, n]; fills ``cache``."""
    pad = _Pad(x.shape[-1] if x.dim() == 3 else p.input(), p.hidden())
    if not pad.needed(x):
        return _qrnn_forward_core(p, x, c0, mode, precision, cache)
    if x.shape[-1] != p.input():
        raise RuntimeError("qrnn_forward: input feature mismatch")
    h = _qrnn_forward_core(pad.qrnn(p), pad.last(x, pad.m, pad.m4), pad.last(c0, pad.n, pad.n4), mode, precision,
                           cache if cache is not None else QrnnCache())
    return h[..., :pad.n].contiguous()


def qrnn_backward(p: QrnnParams, x, c0, cache: QrnnCache, d_h, grads: QrnnGrads, mode="parallel",
                  precision="fp32", want_dc0=True):
    """qrnn_backward (layers.hpp:496-548): accumulates into ``grads``; returns (dx, dc0)."""
    pad = _Pad(p.input(), p.hidden())
    if not pad.needed(x):
        return _qrnn_backward_core(p, x, c0, cache, d_h, grads, mode, precision, want_dc0)
    pp = pad.qrnn(p)
    g4 = QrnnGrads.zeros_like(pp)
    dx, dc0 = _qrnn_backward_core(pp, pad.last(x, pad.m, pad.m4), pad.last(c0, pad.n, pad.n4), cache,
                                  pad.last(d_h, pad.n, pad.n4), g4, mode, precision, want_dc0)
    k = p.window()
    pad.add_rows(grads.W.view(3 * k * pad.n, pad.m), g4.W.view(3 * k * pad.n4, pad.m4), 3 * k, pad.m, pad.m4)
    pad.add_vec(grads.bias, g4.bias, 3)
    return dx[..., :pad.m].contiguous(), None if dc0 is None else dc0[..., :pad.n].contiguous()
