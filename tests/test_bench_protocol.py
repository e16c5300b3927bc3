"""The reference's benchmark protocol pieces used by scripts/bench_kernel.py
(CPU): inputs drawn from Rng(seed).split(1000 + idx) are the reference's
(bench.hpp:134-143, 186; pinned through the oracle's RNG, itself pinned to
test_rng.cpp's known answers) and fnv1a64 is checksum_inputs'
(bench.hpp:69-85)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))


def _fnv_py(data: bytes, h=0xCBF29CE484222325):
    for byte in data:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_fnv1a64_matches_bytewise_definition():
    from paper_1709_04057_b200 import capi
    a = np.arange(37, dtype=np.float32) * 0.37
    b = np.array([1.5, -2.25], dtype=np.float32)
    assert capi.fnv1a64(a, b) == _fnv_py(a.tobytes() + b.tobytes())
    assert capi.fnv1a64() == 0xCBF29CE484222325


def test_bench_inputs_are_the_references(oracle):
    import bench_kernel
    for idx, (T, b, n) in enumerate([(16, 1, 4), (257, 2, 3), (5, 1, 128)]):
        got = bench_kernel.inputs(0, idx, T, b, n)
        ref = oracle.random_recurrence(0, T, b, n, split=1000 + idx)
        for g, r in zip(got, ref):
            assert g.dtype == np.float32 and np.array_equal(g, r)
