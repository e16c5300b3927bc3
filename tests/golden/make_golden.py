"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run here (where /root/reference exists) after ``make -C oracle ref``:

    python tests/golden/make_golden.py

Every output array is produced by the unmodified reference: its own pybind11
module ``linrec`` (proj/bindings/linrec_py.cpp, built into oracle/_ref) for
scan / scan_backward, and the reference's ``linrec::Rng`` (rng.hpp, via the
oracle/_ref C shim) for the bench-distribution inputs.  The fixtures are small
.npz files that travel to the GPU box, where /root/reference does not exist.

The frozen hand-worked vectors of proj/tests/test_recurrence.cpp:75-125 and
:301-316 are stored verbatim alongside (``frozen.npz``).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle.oracle import RefLib, load_reference_module  # noqa: E402


def smoke_instance(rng, T=33, b=2, n=5, dtype=np.float64, lo=-1.0, hi=1.0):
    """proj/tests/python/test_smoke.py:9-13 (numpy default_rng streams)."""
    decays = rng.uniform(lo, hi, size=(T, b, n)).astype(dtype)
    impulses = rng.uniform(-1.0, 1.0, size=(T, b, n)).astype(dtype)
    initial = rng.uniform(-1.0, 1.0, size=(b, n)).astype(dtype)
    return decays, impulses, initial


def main():
    ref = RefLib()
    lr = load_reference_module()
    meta = {"generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/proj (bindings/linrec_py.cpp via oracle/_ref)",
            "cases": {}}

    def save(name, arrays, note):
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrays)
        meta["cases"][name] = {"note": note,
                               "arrays": {k: [list(v.shape), str(v.dtype)] for k, v in arrays.items()}}

    # 1. frozen hand-worked values (test_recurrence.cpp:75-125, :301-316).
    save("frozen", {
        "dyadic_lam": np.array([0.5, 0.25, 0.5, 0.5, 0.25, 0.125]).reshape(3, 1, 2),
        "dyadic_x": np.array([1.5, 2.25, 1.0, 0.5, 0.25, 0.0625]).reshape(3, 1, 2),
        "dyadic_h0": np.array([2.0, 4.0]).reshape(1, 2),
        "dyadic_h": np.array([2.5, 3.25, 2.25, 2.125, 0.8125, 0.328125]).reshape(3, 1, 2),
        "dyadic_dx": np.array([1.625, 1.5625, 1.25, 1.125, 1.0, 1.0]).reshape(3, 1, 2),
        "dyadic_dlam": np.array([3.25, 6.25, 3.125, 3.65625, 2.25, 2.125]).reshape(3, 1, 2),
        "dyadic_dh0": np.array([0.8125, 0.390625]).reshape(1, 2),
        "t1_lam": np.array([0.5, 0.25, 0.75]).reshape(1, 1, 3),
        "t1_x": np.array([1.0, 2.0, 3.0]).reshape(1, 1, 3),
        "t1_h0": np.array([4.0, 8.0, 16.0]).reshape(1, 3),
        "t1_dh": np.array([1.0, -2.0, 0.5]).reshape(1, 1, 3),
        "t1_dlam": np.array([4.0, -16.0, 8.0]).reshape(1, 1, 3),
        "t1_dh0": np.array([0.5, -0.5, 0.375]).reshape(1, 3),
        "two_chunk_h": np.array([1.0, 2.0, 3.0, 4.0]).reshape(4, 1, 1),
        "two_chunk_P": np.array([1.0, 1.0]).reshape(2, 1, 1),
        "two_chunk_R": np.array([2.0, 2.0]).reshape(2, 1, 1),
        "two_chunk_C": np.array([2.0, 4.0]).reshape(2, 1, 1),
        "plan_10_4": np.array([(1, 3), (4, 6), (7, 8), (9, 10)]),
        "plan_3_8": np.array([(1, 1), (2, 2), (3, 3)]),
    }, "hand-worked values frozen in proj/tests/test_recurrence.cpp:27-35,75-125,301-316 and test_smoke.py:93")

    # 2. random instances through the reference's own python API.
    cases = [
        # name, T, b, n, dtype, lam range, seed
        ("smoke_f64", 33, 2, 5, np.float64, (-1.0, 1.0), 7),
        ("smoke_f32", 33, 2, 5, np.float32, (-1.0, 1.0), 7),
        ("t1_w1_f32", 1, 1, 1, np.float32, (0.05, 0.95), 11),
        ("t2_w3_f32", 2, 1, 3, np.float32, (0.05, 0.95), 12),
        ("t257_b2_n4_f32", 257, 2, 4, np.float32, (0.05, 0.95), 13),
        ("t1000_b3_n7_f32", 1000, 3, 7, np.float32, (-1.0, 1.0), 14),
        ("t300_b1_n130_f32", 300, 1, 130, np.float32, (0.05, 0.95), 15),
        ("t513_b2_n64_f32", 513, 2, 64, np.float32, (0.05, 0.95), 16),
        ("t2000_b1_n8_near1_f32", 2000, 1, 8, np.float32, (0.99, 1.0), 17),
        ("t4096_b1_n16_f32", 4096, 1, 16, np.float32, (0.05, 0.95), 18),
        ("t700_b1_n9_f64", 700, 1, 9, np.float64, (-1.0, 1.0), 19),
        ("t129_b2_n66_f64", 129, 2, 66, np.float64, (0.05, 0.95), 20),
    ]
    for name, T, b, n, dt, (lo, hi), seed in cases:
        rng = np.random.default_rng(seed)
        lam, x, h0 = smoke_instance(rng, T, b, n, dt, lo, hi)
        dh = rng.uniform(-1.0, 1.0, size=lam.shape).astype(dt)
        h_serial = lr.scan(lam, x, h0, mode="serial")
        h_par = lr.scan(lam, x, h0, workers=4)
        h_zero = lr.scan(lam, x)  # initial=None -> zeros
        g_serial = lr.scan_backward(lam, h0, h_serial, dh, mode="serial")
        g_par = lr.scan_backward(lam, h0, h_serial, dh, workers=4)
        save(name, {
            "lam": lam, "x": x, "h0": h0, "dh": dh,
            "h_serial": h_serial, "h_parallel_w4": h_par, "h_zero_initial": h_zero,
            "dlam_serial": g_serial[0], "dx_serial": g_serial[1], "dh0_serial": g_serial[2],
            "dlam_parallel_w4": g_par[0], "dx_parallel_w4": g_par[1], "dh0_parallel_w4": g_par[2],
        }, f"numpy default_rng({seed}); lam~U({lo},{hi}); reference linrec.scan/scan_backward")

    # 3. exact identities through the reference (test_recurrence.cpp:185-224).
    T = 50
    lam1 = np.ones((T, 1, 2))
    x1 = np.stack([np.arange(1, T + 1, dtype=np.float64), 2.0 * np.arange(T)], axis=1).reshape(T, 1, 2)
    h01 = np.array([[3.0, -1.0]])
    rng = np.random.default_rng(105)
    x0 = rng.uniform(-5, 5, size=(40, 2, 3))
    h00 = rng.uniform(-5, 5, size=(2, 3))
    save("identities", {
        "ones_lam": lam1, "ones_x": x1, "ones_h0": h01,
        "ones_h": lr.scan(lam1, x1, h01, mode="serial"),
        "zeros_lam": np.zeros_like(x0), "zeros_x": x0, "zeros_h0": h00,
        "zeros_h": lr.scan(np.zeros_like(x0), x0, h00, mode="serial"),
    }, "lambda==1 integer prefix sums and lambda==0 pass-through (test_recurrence.cpp:185-224)")

    # 4. the reference's RNG stream (rng.hpp), KAT of test_rng.cpp:210-223.
    save("rng", {
        "seed42_first3": np.array([ref.rng_first(42, i) for i in range(3)], dtype=np.uint64),
        "split_123_5_f32_u005_095": ref.rng_fill_f32(123, 5, 4096, 0.05, 0.95),
    }, "linrec::Rng draws (rng.hpp:15-71)")

    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(meta["cases"]), "fixtures to", HERE)


if __name__ == "__main__":
    main()
