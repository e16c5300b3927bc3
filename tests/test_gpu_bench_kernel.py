"""scripts/bench_kernel.py (the reference's bench_kernel protocol, bench.hpp:160-244)
on a small grid: the CSV has the reference's header and one serial + one
parallel row per point, the speedup column is serial / parallel, and the
input checksums are the reference's checksum_inputs of the reference's input
stream (recomputed here from the oracle's RNG, pinned to test_rng.cpp)."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "scripts"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_bench_kernel_small_grid(tmp_path, oracle):
    import bench_kernel
    from paper_1709_04057_b200 import capi
    out = tmp_path / "bk.csv"
    rows, sums = bench_kernel.main(["--seq-lens", "16,300", "--features", "4,33", "--batches", "1,2",
                                    "--reps", "3", "--warmup", "1", "--out", str(out)])
    lines = [ln for ln in out.read_text().splitlines() if not ln.startswith("#")]
    assert lines[0] == "T,n,b,workers,impl,events_per_sec,speedup"
    assert len(lines) == 1 + 2 * 8
    for ser, par in zip(lines[1::2], lines[2::2]):
        s, p = ser.split(","), par.split(",")
        assert s[4] == "serial" and p[4] == "parallel" and s[:4] == p[:4]
        assert float(s[6]) == 1.0
        assert float(p[6]) == pytest.approx(float(p[5]) / float(s[5]), rel=1e-6)
    for idx, (T, n, b, csum) in enumerate(sums):
        lam, x, h0 = oracle.random_recurrence(0, T, b, n, split=1000 + idx)
        assert csum == capi.fnv1a64(lam, x, h0)
