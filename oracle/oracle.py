"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  The product package
(paper_1709_04057_b200) never imports it; its CUDA path fails loudly when the
extension is missing instead of falling back here.

Two checkers live behind this module:

* ``Oracle``  -- oracle/liblinrec_oracle.so, the plain-C restatement of
  recurrence.hpp (see oracle/linrec_oracle.c for the file:line map).
* ``RefLib``  -- oracle/_ref/liblinrec_ref.so, the unmodified reference
  compiled from /root/reference by oracle/Makefile (``make -C oracle ref``).
  It travels to the GPU box prebuilt; /root/reference itself does not.

All arrays are C-contiguous ``[T, batch, features]`` (time-major, tensor.hpp:49-75).
"""
from __future__ import annotations

import ctypes as C
import importlib.machinery
import importlib.util
import os
import sysconfig

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblinrec_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_SO = os.path.join(REF_DIR, "liblinrec_ref.so")
REF_PY = os.path.join(REF_DIR, "linrec" + sysconfig.get_config_var("EXT_SUFFIX"))
NATIVE_DIR = os.path.join(REF_DIR, "native")


def _host_cpu_flags():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def native_ref_usable() -> bool:
    """The -march=native reference build (oracle/Makefile) runs here iff this
    host's CPU has every flag of the CPU it was compiled on."""
    try:
        with open(os.path.join(NATIVE_DIR, "cpu_flags.txt")) as f:
            need = set(f.read().split())
    except OSError:
        return False
    return bool(need) and need <= _host_cpu_flags()


def ref_build():
    """(directory, -march) of the reference build the timed baselines load:
    the reference's own -march=native flags where they fit this host."""
    if native_ref_usable() and os.path.exists(os.path.join(NATIVE_DIR, "liblinrec_ref.so")):
        return NATIVE_DIR, "native"
    return REF_DIR, "x86-64-v3"

_i64 = C.c_int64
_vp = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _sfx(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise TypeError(f"oracle: unsupported dtype {dt}")


def max_rel_error(a, b):
    """max|a-b| / max|b| -- tests/support/oracles.hpp:73-82 (normwise)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    max_diff = float(np.max(np.abs(a - b))) if a.size else 0.0
    max_ref = float(np.max(np.abs(b))) if b.size else 0.0
    if max_ref == 0.0:
        return 0.0 if max_diff == 0.0 else float("inf")
    return max_diff / max_ref


def grads_agree(analytic, numeric, rel=1e-5, tiny=1e-7):
    """tests/support/oracles.hpp:64-69."""
    scale = max(abs(analytic), abs(numeric))
    if scale <= tiny:
        return True
    return abs(analytic - numeric) <= rel * scale


class Oracle:
    """The C restatement (oracle/linrec_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        self.lib = lib
        lib.oracle_plan_chunks.restype = _i64
        lib.oracle_plan_chunks.argtypes = [_i64, C.c_int, _vp]
        lib.oracle_predicted_speedup.restype = C.c_double
        lib.oracle_predicted_speedup.argtypes = [C.c_int, _i64]
        for s in ("f32", "f64"):
            getattr(lib, f"oracle_scan_serial_{s}").argtypes = [_vp] * 4 + [_i64] * 2
            getattr(lib, f"oracle_scan_parallel_{s}").argtypes = (
                [_vp] * 4 + [_i64] * 2 + [_vp, _i64] + [_vp] * 3)
            getattr(lib, f"oracle_scan_backward_{s}").argtypes = (
                [_vp] * 7 + [_i64] * 2 + [_vp, _i64])
            getattr(lib, f"oracle_first_nonfinite_{s}").argtypes = [_vp, _i64]
            getattr(lib, f"oracle_first_nonfinite_{s}").restype = _i64
            getattr(lib, f"oracle_rng_fill_{s}").argtypes = [_vp, _vp, _i64, C.c_double, C.c_double]
        lib.oracle_scan_serial_f32_wide.argtypes = [_vp] * 4 + [_i64] * 2
        lib.oracle_scan_backward_f32_wide.argtypes = [_vp] * 7 + [_i64] * 2
        lib.oracle_rng_next_u64.restype = C.c_uint64
        lib.oracle_rng_next_u64.argtypes = [_vp]
        lib.oracle_rng_split.restype = C.c_uint64
        lib.oracle_rng_split.argtypes = [C.c_uint64, C.c_uint64]
        lib.oracle_fnv1a64.restype = C.c_uint64
        lib.oracle_fnv1a64.argtypes = [_vp, C.c_size_t, C.c_uint64]

    # -- plan / cost model --------------------------------------------------
    def plan_chunks(self, T: int, workers: int):
        p = self.lib.oracle_plan_chunks(T, workers, None)
        if p < 0:
            raise RuntimeError("plan_chunks: contract violation")
        b = np.zeros(2 * p, dtype=np.int64)
        self.lib.oracle_plan_chunks(T, workers, _ptr(b))
        return [(int(b[2 * i]), int(b[2 * i + 1])) for i in range(p)]

    def predicted_speedup(self, p: int, T: int) -> float:
        return self.lib.oracle_predicted_speedup(p, T)

    # -- scans ---------------------------------------------------------------
    @staticmethod
    def _shape(a):
        T = a.shape[0]
        W = int(np.prod(a.shape[1:])) if a.ndim > 1 else 1
        return T, W

    def scan_serial(self, lam, x, h0=None):
        lam = np.ascontiguousarray(lam)
        x = np.ascontiguousarray(x, dtype=lam.dtype)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=lam.dtype)
        h = np.empty_like(lam)
        T, W = self._shape(lam)
        getattr(self.lib, f"oracle_scan_serial_{_sfx(lam.dtype)}")(
            _ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, W)
        return h

    def scan_parallel(self, lam, x, h0=None, workers=4, summaries=False):
        lam = np.ascontiguousarray(lam)
        x = np.ascontiguousarray(x, dtype=lam.dtype)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=lam.dtype)
        T, W = self._shape(lam)
        plan = self.plan_chunks(T, workers)
        b = np.asarray(plan, dtype=np.int64).reshape(-1)
        p = len(plan)
        h = np.empty_like(lam)
        P = np.empty((p,) + lam.shape[1:], lam.dtype)
        R = np.empty_like(P)
        Cc = np.empty_like(P)
        getattr(self.lib, f"oracle_scan_parallel_{_sfx(lam.dtype)}")(
            _ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, W, _ptr(b), p,
            _ptr(P), _ptr(R), _ptr(Cc))
        return (h, P, R, Cc) if summaries else h

    def scan_backward(self, lam, h0, h, dh, workers=None):
        """workers=None -> ScanMode::Serial; else the parallel plan."""
        lam = np.ascontiguousarray(lam)
        h = np.ascontiguousarray(h, dtype=lam.dtype)
        dh = np.ascontiguousarray(dh, dtype=lam.dtype)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=lam.dtype)
        T, W = self._shape(lam)
        dlam = np.empty_like(lam)
        dx = np.empty_like(lam)
        dh0 = np.empty(lam.shape[1:], lam.dtype)
        if workers is None:
            b, p = None, 0
        else:
            plan = self.plan_chunks(T, workers)
            b, p = np.asarray(plan, dtype=np.int64).reshape(-1), len(plan)
        getattr(self.lib, f"oracle_scan_backward_{_sfx(lam.dtype)}")(
            _ptr(lam), _ptr(h0), _ptr(h), _ptr(dh), _ptr(dlam), _ptr(dx),
            _ptr(dh0), T, W, _ptr(b), p)
        return dlam, dx, dh0

    def scan_serial_wide(self, lam, x, h0=None):
        """fp64-accumulated serial scan of fp32 data (fp64 error bound)."""
        lam = np.ascontiguousarray(lam, dtype=np.float32)
        x = np.ascontiguousarray(x, dtype=np.float32)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=np.float32)
        h = np.empty(lam.shape, np.float64)
        T, W = self._shape(lam)
        self.lib.oracle_scan_serial_f32_wide(_ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, W)
        return h

    def scan_backward_wide(self, lam, h0, h, dh):
        lam = np.ascontiguousarray(lam, dtype=np.float32)
        h = np.ascontiguousarray(h, dtype=np.float32)
        dh = np.ascontiguousarray(dh, dtype=np.float32)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=np.float32)
        T, W = self._shape(lam)
        dlam = np.empty(lam.shape, np.float64)
        dx = np.empty(lam.shape, np.float64)
        dh0 = np.empty(lam.shape[1:], np.float64)
        self.lib.oracle_scan_backward_f32_wide(
            _ptr(lam), _ptr(h0), _ptr(h), _ptr(dh), _ptr(dlam), _ptr(dx), _ptr(dh0), T, W)
        return dlam, dx, dh0

    # -- GILR / GILR-LSTM layers (oracle/linrec_layers.c) -----------------------
    def _layer_fns(self, dt):
        sfx = _sfx(dt)
        lib = self.lib
        if not getattr(self, f"_layers_{sfx}", False):
            getattr(lib, f"oracle_gilr_forward_{sfx}").argtypes = [_vp] * 6 + [C.c_int] + [_vp] * 3 + [_i64] * 4
            getattr(lib, f"oracle_gilr_backward_{sfx}").argtypes = [_vp] * 4 + [C.c_int] + [_vp] * 10 + [_i64] * 4
            getattr(lib, f"oracle_gilr_lstm_forward_{sfx}").argtypes = [_vp] * 16 + [_i64] * 4
            getattr(lib, f"oracle_gilr_lstm_backward_{sfx}").argtypes = [_vp] * 23 + [_i64] * 4
            getattr(lib, f"oracle_qrnn_forward_{sfx}").argtypes = [_vp] * 7 + [_i64] * 5
            getattr(lib, f"oracle_qrnn_backward_{sfx}").argtypes = [_vp] * 10 + [_i64] * 5
            setattr(self, f"_layers_{sfx}", True)
        return sfx

    def gilr_forward(self, P, x, h0=None, act=0):
        """gilr_forward (layers.hpp:78-100).  P: dict U, V, b_g, b_z.
        Returns h and the cache dict (g, i)."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        n = P["U"].shape[0]
        P = {k: np.ascontiguousarray(v, dtype=dt) for k, v in P.items()}
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=dt)
        h = np.empty((T, b, n), dt)
        cache = {"g": np.empty((T, b, n), dt), "i": np.empty((T, b, n), dt)}
        getattr(self.lib, f"oracle_gilr_forward_{sfx}")(
            _ptr(x), _ptr(P["U"]), _ptr(P["V"]), _ptr(P["b_g"]), _ptr(P["b_z"]), _ptr(h0), act, _ptr(cache["g"]),
            _ptr(cache["i"]), _ptr(h), T, b, m, n)
        return h, cache

    def gilr_backward(self, P, x, h0, cache, h, dh, act=0):
        """gilr_backward (layers.hpp:102-133).  Returns (grads dict, dx, dh0);
        the parameter gradients start at zero."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        n = P["U"].shape[0]
        P = {k: np.ascontiguousarray(v, dtype=dt) for k, v in P.items()}
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=dt)
        g = {k: np.zeros_like(v) for k, v in P.items()}
        dx = np.empty((T, b, m), dt)
        dh0 = np.empty((b, n), dt)
        getattr(self.lib, f"oracle_gilr_backward_{sfx}")(
            _ptr(x), _ptr(P["U"]), _ptr(P["V"]), _ptr(h0), act, _ptr(cache["g"]), _ptr(cache["i"]),
            _ptr(np.ascontiguousarray(h, dtype=dt)), _ptr(np.ascontiguousarray(dh, dtype=dt)), _ptr(g["U"]),
            _ptr(g["V"]), _ptr(g["b_g"]), _ptr(g["b_z"]), _ptr(dx), _ptr(dh0), T, b, m, n)
        return g, dx, dh0

    def gilr_lstm_forward(self, P, x, htil0=None, c0=None):
        """layers.hpp:245-293.  P: dict sU, sV, sbg, sbz, U, V, bias.
        Returns h and the cache dict (sg, si, htil, gates, c)."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        n = P["U"].shape[1]
        P = {k: np.ascontiguousarray(v, dtype=dt) for k, v in P.items()}
        z = np.zeros((b, n), dt)
        htil0 = z if htil0 is None else np.ascontiguousarray(htil0, dtype=dt)
        c0 = z if c0 is None else np.ascontiguousarray(c0, dtype=dt)
        h = np.empty((T, b, n), dt)
        cache = {"sg": np.empty((T, b, n), dt), "si": np.empty((T, b, n), dt), "htil": np.empty((T, b, n), dt),
                 "gates": np.empty((T, b, 4 * n), dt), "c": np.empty((T, b, n), dt)}
        getattr(self.lib, f"oracle_gilr_lstm_forward_{sfx}")(
            _ptr(x), _ptr(P["sU"]), _ptr(P["sV"]), _ptr(P["sbg"]), _ptr(P["sbz"]), _ptr(P["U"]), _ptr(P["V"]),
            _ptr(P["bias"]), _ptr(htil0), _ptr(c0), _ptr(h), _ptr(cache["sg"]), _ptr(cache["si"]),
            _ptr(cache["htil"]), _ptr(cache["gates"]), _ptr(cache["c"]), T, b, m, n)
        return h, cache

    def gilr_lstm_backward(self, P, x, htil0, c0, cache, dh):
        """layers.hpp:295-375.  Returns (grads dict, dx, dhtil0, dc0); the
        parameter gradients start at zero (the reference accumulates)."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        n = P["U"].shape[1]
        P = {k: np.ascontiguousarray(v, dtype=dt) for k, v in P.items()}
        z = np.zeros((b, n), dt)
        htil0 = z if htil0 is None else np.ascontiguousarray(htil0, dtype=dt)
        c0 = z if c0 is None else np.ascontiguousarray(c0, dtype=dt)
        dh = np.ascontiguousarray(dh, dtype=dt)
        g = {k: np.zeros_like(v) for k, v in P.items()}
        dx = np.empty((T, b, m), dt)
        dhtil0 = np.empty((b, n), dt)
        dc0 = np.empty((b, n), dt)
        getattr(self.lib, f"oracle_gilr_lstm_backward_{sfx}")(
            _ptr(x), _ptr(P["sU"]), _ptr(P["sV"]), _ptr(P["U"]), _ptr(P["V"]), _ptr(htil0), _ptr(c0),
            _ptr(cache["sg"]), _ptr(cache["si"]), _ptr(cache["htil"]), _ptr(cache["gates"]), _ptr(cache["c"]),
            _ptr(dh), _ptr(g["sU"]), _ptr(g["sV"]), _ptr(g["sbg"]), _ptr(g["sbz"]), _ptr(g["U"]), _ptr(g["V"]),
            _ptr(g["bias"]), _ptr(dx), _ptr(dhtil0), _ptr(dc0), T, b, m, n)
        return g, dx, dhtil0, dc0

    def qrnn_forward(self, P, x, c0=None):
        """qrnn_forward (layers.hpp:449-494).  P: dict W [k, 3n, m], bias [3n].
        Returns h and the cache dict (gates [T, b, 3n] activated f,o,z; c)."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        W = np.ascontiguousarray(P["W"], dtype=dt)
        k, n3, _ = W.shape
        n = n3 // 3
        bias = np.ascontiguousarray(P["bias"], dtype=dt)
        c0 = np.zeros((b, n), dt) if c0 is None else np.ascontiguousarray(c0, dtype=dt)
        h = np.empty((T, b, n), dt)
        cache = {"gates": np.empty((T, b, 3 * n), dt), "c": np.empty((T, b, n), dt)}
        getattr(self.lib, f"oracle_qrnn_forward_{sfx}")(
            _ptr(x), _ptr(W), _ptr(bias), _ptr(c0), _ptr(h), _ptr(cache["gates"]), _ptr(cache["c"]), T, b, m, n, k)
        return h, cache

    def qrnn_backward(self, P, x, c0, cache, dh):
        """qrnn_backward (layers.hpp:496-548).  Returns (grads dict W, bias;
        dx; dc0); gradients start at zero."""
        x = np.ascontiguousarray(x)
        dt = x.dtype
        sfx = self._layer_fns(dt)
        T, b, m = x.shape
        W = np.ascontiguousarray(P["W"], dtype=dt)
        k, n3, _ = W.shape
        n = n3 // 3
        c0 = np.zeros((b, n), dt) if c0 is None else np.ascontiguousarray(c0, dtype=dt)
        g = {"W": np.zeros_like(W), "bias": np.zeros(3 * n, dt)}
        dx = np.empty((T, b, m), dt)
        dc0 = np.empty((b, n), dt)
        getattr(self.lib, f"oracle_qrnn_backward_{sfx}")(
            _ptr(x), _ptr(W), _ptr(c0), _ptr(cache["gates"]), _ptr(cache["c"]),
            _ptr(np.ascontiguousarray(dh, dtype=dt)), _ptr(g["W"]), _ptr(g["bias"]), _ptr(dx), _ptr(dc0),
            T, b, m, n, k)
        return g, dx, dc0

    def first_nonfinite(self, a):
        a = np.ascontiguousarray(a)
        return int(getattr(self.lib, f"oracle_first_nonfinite_{_sfx(a.dtype)}")(_ptr(a), a.size))

    # -- RNG (rng.hpp) -------------------------------------------------------
    def rng(self, seed: int, split: int | None = None):
        s = seed if split is None else int(self.lib.oracle_rng_split(seed, split))
        return np.array([s, 0], dtype=np.uint64)

    def rng_next(self, state):
        return int(self.lib.oracle_rng_next_u64(_ptr(state)))

    def rng_fill(self, state, shape, lo, hi, dtype=np.float32):
        a = np.empty(shape, dtype)
        getattr(self.lib, f"oracle_rng_fill_{_sfx(dtype)}")(_ptr(state), _ptr(a), a.size, lo, hi)
        return a

    def random_recurrence(self, seed, T, b, n, dtype=np.float32, split=None):
        """bench.hpp:134-143: lam~U(0.05,0.95), x,h0~U(-1,1), one stream."""
        st = self.rng(seed, split)
        lam = self.rng_fill(st, (T, b, n), 0.05, 0.95, dtype)
        x = self.rng_fill(st, (T, b, n), -1.0, 1.0, dtype)
        h0 = self.rng_fill(st, (b, n), -1.0, 1.0, dtype)
        return lam, x, h0

    def fnv1a64(self, *arrays):
        h = 0xCBF29CE484222325
        for a in arrays:
            a = np.ascontiguousarray(a)
            h = int(self.lib.oracle_fnv1a64(_ptr(a), a.nbytes, h))
        return h


class RefLib:
    """The unmodified reference, compiled from /root/reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(path)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        for s in ("f32", "f64"):
            getattr(lib, f"ref_scan_{s}").argtypes = [_vp] * 4 + [_i64] * 3 + [C.c_int, C.c_int] + [_vp] * 3
            getattr(lib, f"ref_scan_backward_{s}").argtypes = [_vp] * 7 + [_i64] * 3 + [C.c_int, C.c_int]
        lib.ref_rng_fill_f32.argtypes = [C.c_uint64, _i64, _vp, _i64, C.c_double, C.c_double]
        lib.ref_rng_first.restype = C.c_uint64
        lib.ref_rng_first.argtypes = [C.c_uint64, C.c_int]
        lib.ref_hardware_workers.restype = C.c_int
        lib.ref_bench_fwd_bwd_f32.argtypes = [_vp] * 4 + [_i64] * 3 + [C.c_int] * 3 + [_vp, _vp]
        lib.ref_bench_serial_f32.argtypes = [_vp] * 4 + [_i64] * 3 + [C.c_int] * 2 + [_vp, _vp]
        lib.ref_gilr_lstm_oracle.argtypes = [_vp] * 11 + [_i64] * 4
        lib.ref_gilr_oracle.argtypes = [_vp] * 7 + [_i64] * 4
        lib.ref_qrnn_oracle.argtypes = [_vp] * 5 + [_i64] * 5

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def scan(self, lam, x, h0=None, mode="parallel", workers=4, summaries=False):
        lam = np.ascontiguousarray(lam)
        x = np.ascontiguousarray(x, dtype=lam.dtype)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=lam.dtype)
        T, b, n = lam.shape
        h = np.empty_like(lam)
        p = min(workers, T)
        P = np.empty((p, b, n), lam.dtype)
        R = np.empty_like(P)
        Cc = np.empty_like(P)
        self._check(getattr(self.lib, f"ref_scan_{_sfx(lam.dtype)}")(
            _ptr(lam), _ptr(x), _ptr(h0), _ptr(h), T, b, n,
            0 if mode == "serial" else 1, workers, _ptr(P), _ptr(R), _ptr(Cc)))
        return (h, P, R, Cc) if summaries else h

    def scan_backward(self, lam, h0, h, dh, mode="parallel", workers=4):
        lam = np.ascontiguousarray(lam)
        h = np.ascontiguousarray(h, dtype=lam.dtype)
        dh = np.ascontiguousarray(dh, dtype=lam.dtype)
        h0 = None if h0 is None else np.ascontiguousarray(h0, dtype=lam.dtype)
        T, b, n = lam.shape
        dlam = np.empty_like(lam)
        dx = np.empty_like(lam)
        dh0 = np.empty((b, n), lam.dtype)
        self._check(getattr(self.lib, f"ref_scan_backward_{_sfx(lam.dtype)}")(
            _ptr(lam), _ptr(h0), _ptr(h), _ptr(dh), _ptr(dlam), _ptr(dx), _ptr(dh0),
            T, b, n, 0 if mode == "serial" else 1, workers))
        return dlam, dx, dh0

    def rng_fill_f32(self, seed, split, count, lo, hi):
        a = np.empty(count, np.float32)
        self.lib.ref_rng_fill_f32(seed, -1 if split is None else split, _ptr(a), count, lo, hi)
        return a

    def rng_first(self, seed, which):
        return int(self.lib.ref_rng_first(seed, which))

    def bench_fwd_bwd(self, lam, x, h0, dh, workers, warmup=1, reps=5):
        """Median seconds of (scan_parallel, scan_backward(Parallel)) on the
        host cores, reference bench protocol (bench.hpp:93-107)."""
        lam, x, h0, dh = (np.ascontiguousarray(a, dtype=np.float32) for a in (lam, x, h0, dh))
        T, b, n = lam.shape
        f = C.c_double(0.0)
        bw = C.c_double(0.0)
        self._check(self.lib.ref_bench_fwd_bwd_f32(
            _ptr(lam), _ptr(x), _ptr(h0), _ptr(dh), T, b, n, workers, warmup, reps,
            C.byref(f), C.byref(bw)))
        return f.value, bw.value

    def bench_serial(self, lam, x, h0, dh, warmup=0, reps=1):
        """Median seconds of (scan_serial, scan_backward(Serial)): the
        reference's 1-core path, same protocol."""
        lam, x, h0, dh = (np.ascontiguousarray(a, dtype=np.float32) for a in (lam, x, h0, dh))
        T, b, n = lam.shape
        f = C.c_double(0.0)
        bw = C.c_double(0.0)
        self._check(self.lib.ref_bench_serial_f32(
            _ptr(lam), _ptr(x), _ptr(h0), _ptr(dh), T, b, n, warmup, reps, C.byref(f), C.byref(bw)))
        return f.value, bw.value

    def gilr_lstm_oracle(self, P, x, htil0, c0):
        """The reference's per-step GILR-LSTM (layer_oracles.hpp:52-82), fp64."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        T, b, m = x.shape
        n = P["U"].shape[1]
        P = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in P.items()}
        h = np.empty((T, b, n))
        self._check(self.lib.ref_gilr_lstm_oracle(
            _ptr(x), _ptr(P["sU"]), _ptr(P["sV"]), _ptr(P["sbg"]), _ptr(P["sbz"]), _ptr(P["U"]), _ptr(P["V"]),
            _ptr(P["bias"]), _ptr(np.ascontiguousarray(htil0, dtype=np.float64)),
            _ptr(np.ascontiguousarray(c0, dtype=np.float64)), _ptr(h), T, b, m, n))
        return h

    def qrnn_oracle(self, P, x, c0):
        """The reference's per-step QRNN (layer_oracles.hpp:84-114), fp64."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        T, b, m = x.shape
        W = np.ascontiguousarray(P["W"], dtype=np.float64)
        k, n3, _ = W.shape
        h = np.empty((T, b, n3 // 3))
        self._check(self.lib.ref_qrnn_oracle(
            _ptr(x), _ptr(W), _ptr(np.ascontiguousarray(P["bias"], dtype=np.float64)),
            _ptr(np.ascontiguousarray(c0, dtype=np.float64)), _ptr(h), T, b, m, n3 // 3, k))
        return h

    def hardware_workers(self):
        return int(self.lib.ref_hardware_workers())


def load_reference_module(ref_dir: str = REF_DIR):
    """The reference's own pybind11 module ``linrec`` (bindings/linrec_py.cpp)
    built into oracle/_ref (or ref_build()'s directory).  Loaded without
    touching sys.modules so it never shadows the product module of the same
    name."""
    path = os.path.join(ref_dir, os.path.basename(REF_PY))
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
    loader = importlib.machinery.ExtensionFileLoader("linrec", path)
    spec = importlib.util.spec_from_file_location("linrec", path, loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


def qrnn_params(rng, m, n, k, dtype=np.float64, gate_bias=1.0):
    """Random QRNN parameters shaped like qrnn_init (layers.hpp:411-422):
    k taps W_s ~ U(+-1/sqrt(m k)) packed [k, 3n, m], bias = gate_bias on f."""
    s = 1.0 / np.sqrt(m * k)
    bias = np.zeros(3 * n)
    bias[:n] = gate_bias
    return {"W": rng.uniform(-s, s, (k, 3 * n, m)).astype(dtype), "bias": bias.astype(dtype)}


def gilr_lstm_params(rng, m, n, dtype=np.float64, gate_bias=1.0):
    """Random GILR-LSTM parameters shaped like gilr_lstm_init (layers.hpp:165-175):
    U ~ U(+-1/sqrt(n)), V ~ U(+-1/sqrt(m)), gate bias on the f block."""
    sm, sn = 1.0 / np.sqrt(m), 1.0 / np.sqrt(n)
    bias = np.zeros(4 * n)
    bias[:n] = gate_bias
    P = {"sU": rng.uniform(-sm, sm, (n, m)), "sV": rng.uniform(-sm, sm, (n, m)),
         "sbg": np.full(n, gate_bias), "sbz": np.zeros(n),
         "U": rng.uniform(-sn, sn, (4 * n, n)), "V": rng.uniform(-sm, sm, (4 * n, m)), "bias": bias}
    return {k: v.astype(dtype) for k, v in P.items()}
