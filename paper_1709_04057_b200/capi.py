"""ctypes binding of the C ABI (include/linrec_cuda.h) for device-pointer use.

This is the boundary a Python host (bench.py, the sharded driver, tests) uses
to call the sm_100a kernels on buffers it already owns -- e.g. torch CUDA
tensors -- on a given CUDA stream.  It loads ``liblinrec_cuda.so`` from this
package directory and raises ``ImportError`` when it is missing: there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LINREC_LIB_PATH") or os.path.join(HERE, "liblinrec_cuda.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "linrec_cuda.h")

SERIAL = 0
PARALLEL = 1
KERNEL_AUTO = 0
KERNEL_REGISTER = 1

OK, ERR_SHAPE, ERR_DTYPE, ERR_VALUE, ERR_CUDA, ERR_NONFINITE, ERR_INTERNAL = range(7)

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int


class Exchange(C.Structure):
    """linrec_exchange_t: one direction of the fused peer-memory carry exchange."""
    _fields_ = [("mboxes", _vp), ("world", _int), ("rank", _int), ("epoch", C.c_uint64),
                ("consumers_first", _int), ("consumers_last", _int),
                ("sources_first", _int), ("sources_last", _int), ("sources_step", _int), ("zero_a", _int)]


class LinrecError(RuntimeError):
    """A non-zero linrec_status; ``code`` is the status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "linrec has no CPU path")
    lib = C.CDLL(LIB_PATH)
    lib.linrec_last_error.restype = C.c_char_p
    lib.linrec_abi_version.restype = _int
    lib.linrec_device_count.restype = _int
    lib.linrec_workspace_bytes.restype = C.c_size_t
    lib.linrec_workspace_bytes.argtypes = [_i64, _i64, _int]
    lib.linrec_workspace_create.argtypes = [C.POINTER(_vp), _int]
    lib.linrec_workspace_destroy.argtypes = [_vp]
    lib.linrec_set_kernel_policy.argtypes = [_int]
    lib.linrec_device_malloc.argtypes = [C.POINTER(_vp), C.c_size_t, _int, _vp]
    lib.linrec_device_free.argtypes = [_vp, _int, _vp]
    for s in ("f32", "f64"):
        getattr(lib, f"linrec_scan_{s}").argtypes = [_vp] * 4 + [_i64, _i64, _int, _vp, _vp]
        getattr(lib, f"linrec_scan_backward_{s}").argtypes = [_vp] * 7 + [_i64, _i64, _int, _vp, _vp]
        getattr(lib, f"linrec_scan_backward_segment_{s}").argtypes = [_vp] * 9 + [_i64, _i64, _int, _vp, _vp]
        getattr(lib, f"linrec_scan_host_{s}").argtypes = [_vp] * 4 + [_i64, _i64, _int, _int]
        getattr(lib, f"linrec_scan_backward_host_{s}").argtypes = [_vp] * 7 + [_i64, _i64, _int, _int]
        getattr(lib, f"linrec_first_nonfinite_{s}").argtypes = [_vp, _i64, C.POINTER(_i64), _vp]
        getattr(lib, f"linrec_screen_finite_{s}").argtypes = [_vp, _i64, _i64, _i64, C.c_char_p, _vp]
        getattr(lib, f"linrec_segment_scan_{s}").argtypes = [_vp] * 6 + [_i64, _i64, _vp, _vp]
        getattr(lib, f"linrec_segment_scan_backward_{s}").argtypes = [_vp] * 10 + [_i64, _i64, _vp, _vp]
        getattr(lib, f"linrec_compose_carries_{s}").argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp]
        getattr(lib, f"linrec_segment_fixup_{s}").argtypes = [_vp] * 4 + [_i64, _i64, _i64, _vp]
        getattr(lib, f"linrec_segment_fixup_backward_{s}").argtypes = [_vp] * 8 + [_i64, _i64, _i64, _vp]
    lib.linrec_gemm_f32.argtypes = [_vp, _int, _i64, _vp, _int, _i64, _vp, _i64, _i64, _i64, _i64, _int, _int,
                                    _int, _vp, _vp]
    lib.linrec_gemm_splits.argtypes = [_i64, _i64, _i64]
    lib.linrec_p2p_mailbox_bytes.restype = C.c_size_t
    lib.linrec_p2p_mailbox_bytes.argtypes = [_i64, _int]
    lib.linrec_ipc_alloc.argtypes = [C.c_size_t, C.POINTER(_vp), C.c_char_p]
    lib.linrec_ipc_open.argtypes = [C.c_char_p, C.POINTER(_vp)]
    lib.linrec_ipc_close.argtypes = [_vp]
    lib.linrec_ipc_free.argtypes = [_vp]
    lib.linrec_p2p_publish_f32.argtypes = [_vp, _i64, _int, _int, _int, C.c_uint64, _vp, _int, _int, _vp]
    lib.linrec_p2p_compose_f32.argtypes = [_i64, _int, _int, _int, C.c_uint64, _vp, _vp, _i64, _i64, _i64, _vp,
                                           _vp, _vp]
    for s_ in ("f32", "f64"):
        getattr(lib, f"linrec_scan_plan_{s_}").argtypes = [_vp] * 4 + [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp]
        getattr(lib, f"linrec_scan_backward_plan_{s_}").argtypes = [_vp] * 7 + [_i64, _i64, _vp, _i64, _vp]
    lib.linrec_scan_kernel_count.argtypes = [_i64, _i64, _int, _int, _int]
    lib.linrec_scan_kernel_name.restype = C.c_char_p
    lib.linrec_scan_kernel_name.argtypes = [_i64, _i64, _int, _int, _int]
    _ex = C.POINTER(Exchange)
    lib.linrec_segment_scan_exchange_f32.argtypes = [_vp] * 6 + [_i64, _i64, _ex, _vp, _vp]
    lib.linrec_segment_scan_backward_exchange_f32.argtypes = [_vp] * 10 + [_i64, _i64, _ex, _vp, _vp]
    lib.linrec_segment_fixup_exchange_f32.argtypes = [_vp] * 4 + [_i64, _i64, _i64, _ex, _vp]
    lib.linrec_segment_fixup_backward_exchange_f32.argtypes = [_vp] * 8 + [_i64, _i64, _i64, _ex, _vp]
    lib.linrec_gemm_scratch_bytes.restype = C.c_size_t
    lib.linrec_gemm_scratch_bytes.argtypes = [_i64, _i64, _int]
    lib.linrec_segment_prod_rows.restype = _i64
    lib.linrec_segment_prod_rows.argtypes = [_i64, _i64, _int, _int]
    lib.linrec_segment_tile_rows.restype = _i64
    lib.linrec_segment_tile_rows.argtypes = [_i64, _i64, _int, _int]
    for s_ in ("f32", "f64"):
        getattr(lib, f"linrec_scan_host_columns_{s_}").argtypes = [_vp] * 4 + [_i64] * 4 + [_int, _int]
        getattr(lib, f"linrec_scan_backward_host_columns_{s_}").argtypes = [_vp] * 7 + [_i64] * 4 + [_int, _int]
        getattr(lib, f"linrec_scan_host_multi_{s_}").argtypes = [_vp] * 4 + [_i64, _i64, _int, C.POINTER(_int), _int]
        getattr(lib, f"linrec_scan_backward_host_multi_{s_}").argtypes = [_vp] * 7 + [_i64, _i64, _int,
                                                                                     C.POINTER(_int), _int]
    lib.linrec_column_block.argtypes = [_i64, _int, _int, C.POINTER(_i64), C.POINTER(_i64)]
    lib.linrec_scan_backward_gated_f32.argtypes = [_vp] * 8 + [_i64, _i64, _int, _vp, _vp]
    lib.linrec_fnv1a64.restype = C.c_uint64
    lib.linrec_fnv1a64.argtypes = [_vp, C.c_size_t, C.c_uint64]
    return lib


lib = _load()


def declared_symbols(header: str = HEADER):
    """Function names declared in include/linrec_cuda.h."""
    with open(header) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(linrec_[a-z0-9_]+)\s*\(", text)))


def set_kernel_policy(policy: int):
    """KERNEL_AUTO (TMA persistent kernels where eligible) or KERNEL_REGISTER."""
    check(lib.linrec_set_kernel_policy(policy))


def check(rc: int):
    if rc != OK:
        raise LinrecError(rc, lib.linrec_last_error().decode())


def _sfx(dtype_bytes: int) -> str:
    if dtype_bytes == 4:
        return "f32"
    if dtype_bytes == 8:
        return "f64"
    raise TypeError("decays must be float32 or float64")


def scan(lam, x, h0, h, T, W, mode=PARALLEL, dtype_bytes=4, ws=None, stream=0):
    """Device pointers (ints) -> linrec_scan_{f32,f64}."""
    check(getattr(lib, f"linrec_scan_{_sfx(dtype_bytes)}")(lam, x, h0, h, T, W, mode, ws, stream))


def scan_backward(lam, h0, h, dh, dlam, dx, dh0, T, W, mode=PARALLEL, dtype_bytes=4, ws=None, stream=0):
    check(getattr(lib, f"linrec_scan_backward_{_sfx(dtype_bytes)}")(
        lam, h0, h, dh, dlam, dx, dh0, T, W, mode, ws, stream))


def scan_backward_segment(lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W, mode=PARALLEL,
                          dtype_bytes=4, ws=None, stream=0):
    check(getattr(lib, f"linrec_scan_backward_segment_{_sfx(dtype_bytes)}")(
        lam, h0, h, dh, lam_next, g_next, dlam, dx, dh0, T, W, mode, ws, stream))


def scan_host(lam, x, h0, h, T, W, mode=PARALLEL, dtype_bytes=4, device=0):
    """Host pointers -> linrec_scan_host_* (pipelined H2D / scan / D2H)."""
    check(getattr(lib, f"linrec_scan_host_{_sfx(dtype_bytes)}")(lam, x, h0, h, T, W, mode, device))


def scan_backward_host(lam, h0, h, dh, dlam, dx, dh0, T, W, mode=PARALLEL, dtype_bytes=4, device=0):
    check(getattr(lib, f"linrec_scan_backward_host_{_sfx(dtype_bytes)}")(
        lam, h0, h, dh, dlam, dx, dh0, T, W, mode, device))


# ---- channel sharding of host arrays ----------------------------------------
def scan_host_columns(lam, x, h0, h, T, W, c0, c1, mode=PARALLEL, dtype_bytes=4, device=0):
    """Columns [c0, c1) of host [T][W] arrays on `device` (2-D staged copies)."""
    check(getattr(lib, f"linrec_scan_host_columns_{_sfx(dtype_bytes)}")(lam, x, h0, h, T, W, c0, c1, mode, device))


def scan_backward_host_columns(lam, h0, h, dh, dlam, dx, dh0, T, W, c0, c1, mode=PARALLEL, dtype_bytes=4,
                               device=0):
    check(getattr(lib, f"linrec_scan_backward_host_columns_{_sfx(dtype_bytes)}")(
        lam, h0, h, dh, dlam, dx, dh0, T, W, c0, c1, mode, device))


def _devs(devices):
    devices = list(devices)
    return (_int * len(devices))(*devices), len(devices)


def scan_host_multi(lam, x, h0, h, T, W, devices, mode=PARALLEL, dtype_bytes=4):
    """Channel-sharded scan of host [T][W] arrays over `devices` (one host thread each)."""
    d, n = _devs(devices)
    check(getattr(lib, f"linrec_scan_host_multi_{_sfx(dtype_bytes)}")(lam, x, h0, h, T, W, mode, d, n))


def scan_backward_host_multi(lam, h0, h, dh, dlam, dx, dh0, T, W, devices, mode=PARALLEL, dtype_bytes=4):
    d, n = _devs(devices)
    check(getattr(lib, f"linrec_scan_backward_host_multi_{_sfx(dtype_bytes)}")(
        lam, h0, h, dh, dlam, dx, dh0, T, W, mode, d, n))


FNV_OFFSET = 0xCBF29CE484222325


def fnv1a64(*arrays, h=FNV_OFFSET) -> int:
    """checksum_inputs (bench.hpp:69-85): FNV-1a 64 over the arrays' bytes in order."""
    for a in arrays:
        h = int(lib.linrec_fnv1a64(a.ctypes.data, a.nbytes, h))
    return h


def column_block(W, n, d):
    """Columns [c0, c1) of device d of n under channel sharding."""
    c0, c1 = _i64(), _i64()
    check(lib.linrec_column_block(W, n, d, C.byref(c0), C.byref(c1)))
    return int(c0.value), int(c1.value)


def first_nonfinite(v, n, dtype_bytes=4, stream=0) -> int:
    out = _i64(-1)
    check(getattr(lib, f"linrec_first_nonfinite_{_sfx(dtype_bytes)}")(v, n, C.byref(out), stream))
    return int(out.value)


def screen_finite(v, T, batch, features, name, dtype_bytes=4, stream=0):
    """screen_finite (recurrence.hpp:133-155): raises LinrecError (code
    ERR_NONFINITE) with the reference's message; T = 0 for a [batch, features]
    tensor."""
    check(getattr(lib, f"linrec_screen_finite_{_sfx(dtype_bytes)}")(v, T, batch, features, name.encode(), stream))


# ---- sequence sharding (see include/linrec_cuda.h) ---------------------------
def segment_prod_rows(T, W, backward=False, dtype_bytes=4) -> int:
    return int(lib.linrec_segment_prod_rows(T, W, dtype_bytes, 1 if backward else 0))


def segment_tile_rows(T, W, backward=False, dtype_bytes=4) -> int:
    return int(lib.linrec_segment_tile_rows(T, W, dtype_bytes, 1 if backward else 0))


def segment_scan(lam, x, h0, h, seg_prod, agg, T, W, dtype_bytes=4, ws=None, stream=0):
    check(getattr(lib, f"linrec_segment_scan_{_sfx(dtype_bytes)}")(lam, x, h0, h, seg_prod, agg, T, W, ws, stream))


def segment_scan_backward(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, dtype_bytes=4,
                          ws=None, stream=0):
    check(getattr(lib, f"linrec_segment_scan_backward_{_sfx(dtype_bytes)}")(
        lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ws, stream))


def compose_carries(aggs, first, last, step, seed, out, W, dtype_bytes=4, stream=0):
    check(getattr(lib, f"linrec_compose_carries_{_sfx(dtype_bytes)}")(aggs, first, last, step, seed, out, W, stream))


def segment_fixup(lam, h, seg_prod, c_in, T, W, tile_rows, dtype_bytes=4, stream=0):
    check(getattr(lib, f"linrec_segment_fixup_{_sfx(dtype_bytes)}")(lam, h, seg_prod, c_in, T, W, tile_rows, stream))


def segment_fixup_backward(lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, tile_rows, dtype_bytes=4,
                           stream=0):
    check(getattr(lib, f"linrec_segment_fixup_backward_{_sfx(dtype_bytes)}")(
        lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, tile_rows, stream))


def scan_kernel_count(T, W, backward=False, mode=PARALLEL, dtype_bytes=4) -> int:
    """Kernels one scan (or scan_backward) call launches for this shape."""
    return int(lib.linrec_scan_kernel_count(T, W, dtype_bytes, 1 if backward else 0, mode))


def scan_kernel_name(T, W, backward=False, mode=PARALLEL, dtype_bytes=4) -> str:
    """Kernel family of that call: serial, cluster, local, tma or chained."""
    r = lib.linrec_scan_kernel_name(T, W, dtype_bytes, 1 if backward else 0, mode)
    if r is None:
        raise LinrecError(ERR_VALUE, "scan_kernel_name: invalid arguments")
    return r.decode()


# ---- the reference's chunked scan with an explicit plan ---------------------
def _bounds(plan):
    flat = (C.c_int64 * (2 * len(plan)))(*[v for se in plan for v in se])
    return flat, len(plan)


def scan_plan(lam, x, h0, h, T, W, plan, P=None, R=None, Cs=None, dtype_bytes=4, stream=0):
    """plan: [(start, end), ...] 1-based inclusive (linrec.plan_chunks)."""
    b, p = _bounds(plan)
    check(getattr(lib, f"linrec_scan_plan_{_sfx(dtype_bytes)}")(lam, x, h0, h, T, W, b, p, P, R, Cs, stream))


def scan_backward_plan(lam, h0, h, dh, dlam, dx, dh0, T, W, plan, dtype_bytes=4, stream=0):
    b, p = _bounds(plan)
    check(getattr(lib, f"linrec_scan_backward_plan_{_sfx(dtype_bytes)}")(lam, h0, h, dh, dlam, dx, dh0, T, W, b, p,
                                                                         stream))


# the same with the carry exchange fused into the stitch kernels (fp32; ex: Exchange)
def segment_scan_exchange(lam, x, h0, h, seg_prod, agg, T, W, ex, ws=None, stream=0):
    check(lib.linrec_segment_scan_exchange_f32(lam, x, h0, h, seg_prod, agg, T, W, C.byref(ex), ws, stream))


def segment_scan_backward_exchange(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg, T, W, ex, ws=None,
                                   stream=0):
    check(lib.linrec_segment_scan_backward_exchange_f32(lam, hprev, h, dh, lam_next, dlam, dx, dh0, seg_prod, agg,
                                                        T, W, C.byref(ex), ws, stream))


def segment_fixup_exchange(lam, h, seg_prod, c_in, T, W, tile_rows, ex, stream=0):
    check(lib.linrec_segment_fixup_exchange_f32(lam, h, seg_prod, c_in, T, W, tile_rows, C.byref(ex), stream))


def segment_fixup_backward_exchange(lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W, tile_rows, ex,
                                    stream=0):
    check(lib.linrec_segment_fixup_backward_exchange_f32(lam, hprev, h, lam_next, seg_prod, y_in, dlam, dx, T, W,
                                                         tile_rows, C.byref(ex), stream))


PREC_FP32 = 0
PREC_TF32 = 1


def gemm(A, a_mn, lda, B, b_mn, ldb, C, ldc, M, N, K, accumulate=False, precision=PREC_FP32, k_splits=1,
         scratch=None, stream=0):
    """tcgen05 GEMM (device pointers), see include/linrec_cuda.h."""
    check(lib.linrec_gemm_f32(A, int(a_mn), lda, B, int(b_mn), ldb, C, ldc, M, N, K, int(accumulate), precision,
                              k_splits, scratch, stream))


def gemm_splits(M, N, K) -> int:
    return int(lib.linrec_gemm_splits(M, N, K))


def gemm_scratch_bytes(M, N, k_splits) -> int:
    return int(lib.linrec_gemm_scratch_bytes(M, N, k_splits))


class Workspace:
    """Explicit look-back workspace (one per concurrent stream)."""

    def __init__(self, device: int = 0):
        self.handle = _vp()
        check(lib.linrec_workspace_create(C.byref(self.handle), device))

    def close(self):
        if self.handle:
            lib.linrec_workspace_destroy(self.handle)
            self.handle = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
