"""Pin the CPU oracle (oracle/linrec_oracle.c) before trusting it.

The oracle must reproduce, bit for bit, (1) the reference's frozen hand-worked
vectors (proj/tests/test_recurrence.cpp) and (2) the fixtures produced by the
reference itself (tests/golden/make_golden.py).  CPU only.
"""
import numpy as np
import pytest

from conftest import RANDOM_CASES, load_golden


def test_frozen_dyadic_forward_backward(oracle):
    g = load_golden("frozen")
    for dt in (np.float64, np.float32):
        lam, x, h0 = (g[k].astype(dt) for k in ("dyadic_lam", "dyadic_x", "dyadic_h0"))
        h = oracle.scan_serial(lam, x, h0)
        assert np.array_equal(h, g["dyadic_h"].astype(dt))
        dh = np.ones_like(lam)
        for workers in (None, 2):  # ScanMode::Serial / Parallel (test_recurrence.cpp:117)
            dlam, dx, dh0 = oracle.scan_backward(lam, h0, h, dh, workers=workers)
            assert np.array_equal(dx, g["dyadic_dx"].astype(dt))
            assert np.array_equal(dlam, g["dyadic_dlam"].astype(dt))
            assert np.array_equal(dh0, g["dyadic_dh0"].astype(dt))


def test_frozen_t1_backward(oracle):
    g = load_golden("frozen")
    h = oracle.scan_serial(g["t1_lam"], g["t1_x"], g["t1_h0"])
    dlam, dx, dh0 = oracle.scan_backward(g["t1_lam"], g["t1_h0"], h, g["t1_dh"], workers=2)
    assert np.array_equal(dlam, g["t1_dlam"])
    assert np.array_equal(dx, g["t1_dh"])
    assert np.array_equal(dh0, g["t1_dh0"])


def test_two_chunk_summaries(oracle):
    g = load_golden("frozen")
    lam = np.ones((4, 1, 1))
    h, P, R, C = oracle.scan_parallel(lam, np.ones_like(lam), np.zeros((1, 1)), workers=2, summaries=True)
    for k, v in (("h", h), ("P", P), ("R", R), ("C", C)):
        assert np.array_equal(v, g[f"two_chunk_{k}"]), k


def test_plan_chunks(oracle):
    g = load_golden("frozen")
    assert oracle.plan_chunks(10, 4) == [tuple(r) for r in g["plan_10_4"].tolist()]
    assert oracle.plan_chunks(3, 8) == [tuple(r) for r in g["plan_3_8"].tolist()]
    for T in (1, 2, 3, 7, 8, 100, 65536):  # test_recurrence.cpp:37-60
        for w in (1, 2, 3, 4, 7, 8, 16, 17):
            plan = oracle.plan_chunks(T, w)
            assert len(plan) == min(w, T)
            assert plan[0][0] == 1 and plan[-1][1] == T
            lens = [e - s + 1 for s, e in plan]
            assert max(lens) - min(lens) <= 1 and lens == sorted(lens, reverse=True)
            assert all(e + 1 == s2 for (s, e), (s2, _) in zip(plan, plan[1:]))
    with pytest.raises(RuntimeError):
        oracle.plan_chunks(0, 4)
    with pytest.raises(RuntimeError):
        oracle.plan_chunks(4, 0)


def test_predicted_speedup(oracle):  # test_smoke.py:96-99
    assert oracle.predicted_speedup(1, 1000) == pytest.approx(1 / 3)
    assert 0.95 <= oracle.predicted_speedup(3, 100000) <= 1.0
    assert oracle.predicted_speedup(8, 1 << 20) > 2.0


@pytest.mark.parametrize("name", RANDOM_CASES)
def test_oracle_matches_reference_fixtures_bitwise(oracle, name):
    g = load_golden(name)
    lam, x, h0, dh = g["lam"], g["x"], g["h0"], g["dh"]
    assert np.array_equal(oracle.scan_serial(lam, x, h0), g["h_serial"])
    assert np.array_equal(oracle.scan_parallel(lam, x, h0, workers=4), g["h_parallel_w4"])
    h = g["h_serial"]
    for tag, workers in (("serial", None), ("parallel_w4", 4)):
        dlam, dx, dh0 = oracle.scan_backward(lam, h0, h, dh, workers=workers)
        assert np.array_equal(dlam, g[f"dlam_{tag}"])
        assert np.array_equal(dx, g[f"dx_{tag}"])
        assert np.array_equal(dh0, g[f"dh0_{tag}"])


@pytest.mark.parametrize("name", RANDOM_CASES)
def test_oracle_within_fp64_bound(oracle, name):
    """test_smoke.py:27-37: f32 <= 1e-5 / f64 <= 1e-12 normwise vs fp64."""
    from oracle.oracle import max_rel_error
    g = load_golden(name)
    if g["lam"].dtype != np.float32:
        pytest.skip("fp64 case")
    wide = oracle.scan_serial_wide(g["lam"], g["x"], g["h0"])
    assert max_rel_error(g["h_serial"], wide) < 1e-5


def test_identities_exact(oracle):
    g = load_golden("identities")
    assert np.array_equal(oracle.scan_serial(g["ones_lam"], g["ones_x"], g["ones_h0"]), g["ones_h"])
    assert np.array_equal(oracle.scan_serial(g["zeros_lam"], g["zeros_x"], g["zeros_h0"]), g["zeros_x"])
    run = np.cumsum(g["ones_x"], axis=0) + g["ones_h0"]
    assert np.array_equal(g["ones_h"], run)


def test_rng_kat(oracle):
    g = load_golden("rng")
    st = oracle.rng(42)
    assert [oracle.rng_next(st) for _ in range(3)] == [int(v) for v in g["seed42_first3"]]
    assert [0xBDD732262FEB6E95, 0x28EFE333B266F103, 0x47526757130F9F52] == [int(v) for v in g["seed42_first3"]]
    assert int(oracle.lib.oracle_rng_split(42, 7)) == 0x583E77C90AF5C134  # test_rng.cpp:219
    st = oracle.rng(123, 5)
    assert np.array_equal(oracle.rng_fill(st, (4096,), 0.05, 0.95), g["split_123_5_f32_u005_095"])


def test_oracle_against_compiled_reference_when_present(oracle):
    """Live check against oracle/_ref (the reference compiled from source)."""
    import os
    from oracle.oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        for (T, b, n) in [(1, 1, 1), (64, 3, 5), (1000, 2, 33)]:
            lam = rng.uniform(-1, 1, (T, b, n)).astype(dt)
            x = rng.uniform(-1, 1, (T, b, n)).astype(dt)
            h0 = rng.uniform(-1, 1, (b, n)).astype(dt)
            assert np.array_equal(oracle.scan_serial(lam, x, h0), ref.scan(lam, x, h0, mode="serial"))
            for w in (1, 3, 8):
                assert np.array_equal(oracle.scan_parallel(lam, x, h0, workers=w), ref.scan(lam, x, h0, workers=w))
