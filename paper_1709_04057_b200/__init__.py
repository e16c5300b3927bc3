"""B200-native parallel linear recurrence (arXiv 1709.04057).

    h_t = lam_t * h_{t-1} + x_t      and its reverse-time gradient scan,

on hand-written sm_100a kernels behind a C ABI (include/linrec_cuda.h).

* ``linrec``    -- drop-in for the reference's pybind11 module
                   (proj/bindings/linrec_py.cpp): scan, scan_backward,
                   plan_chunks, predicted_speedup, hardware_workers.
* ``capi``      -- ctypes binding of the C ABI (device / host pointers).
* ``torch_ops`` -- torch CUDA tensors on the current stream (+ autograd).
* ``sharded``   -- sequence / channel sharding across GPUs.

Importing fails loudly if the native library is missing; there is no CPU
compute path.
"""
import os as _os
import sys as _sys

_HERE = _os.path.dirname(_os.path.abspath(__file__))

from . import capi  # noqa: E402  (raises ImportError without liblinrec_cuda.so)

if _HERE not in _sys.path:
    _sys.path.insert(0, _HERE)
import linrec  # noqa: E402  the pybind11 module built next to this file

if _os.path.dirname(_os.path.abspath(linrec.__file__)) != _HERE:
    raise ImportError(f"linrec resolved to {linrec.__file__}, expected the build in {_HERE}")

__all__ = ["linrec", "capi"]
