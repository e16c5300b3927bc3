"""The C++ drop-in headers (include/linrec/cuda_scan.hpp, cuda_layers.hpp)
exercised by a C++ program the way a reference C++ call site would use them
(tests/cpp/test_cuda_api.cpp, built by `make cpp-tests`)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_api_program():
    exe = os.path.join(ROOT, "build", "test_cuda_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpp-tests"], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    if out.returncode == 2 and "no CUDA device" in out.stderr:
        pytest.skip("no CUDA device")
    assert out.returncode == 0, out.stderr[-3000:]
    assert "ALL OK" in out.stdout


@pytest.mark.parametrize("world,T,W,lo,hi", [(2, 1 << 20, 128, 0.05, 0.95), (3, 30001, 64, 0.99, 1.0),
                                             (2, 9000, 384, -1.0, 1.0)])
def test_cpp_sharded_ranks(oracle, tmp_path, world, T, W, lo, hi):
    """The multi-GPU C ABI from C++ (tests/cpp/test_sharded.cpp over
    include/linrec/cuda_sharded.hpp): `world` processes share the GPU,
    exchange mailbox handles through files and run 3 sequence-sharded
    forward + backward steps; their rows match the unsharded oracle (1e-5
    normwise, test_smoke.py:35) -- the C4 shape at full T included."""
    import numpy as np
    from oracle.oracle import max_rel_error
    exe = os.path.join(ROOT, "build", "test_sharded")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpp-tests"], check=True, capture_output=True)
    rng = np.random.default_rng(T + W)
    lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (W,)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    for name, a in (("lam", lam), ("x", x), ("h0", h0), ("dh", dh)):
        a.tofile(tmp_path / f"{name}.bin")
    procs = [subprocess.Popen([exe, str(tmp_path), str(r), str(world), str(T), str(W), "3"],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        if p.returncode == 2 and "no CUDA device" in e:
            pytest.skip("no CUDA device")
        assert p.returncode == 0, e[-3000:]
    h_ref = oracle.scan_serial(lam, x, h0)
    g = oracle.scan_backward_wide(lam, h0, h_ref, dh)
    h_wide = oracle.scan_serial_wide(lam, x, h0)
    base, rem = divmod(T, world)
    for r in range(world):
        s = r * base + min(r, rem)
        e = s + base + (1 if r < rem else 0)
        rd = lambda n: np.fromfile(tmp_path / f"out_{r}_{n}.bin", dtype=np.float32).reshape(-1, W)  # noqa: E731
        assert max_rel_error(rd("h"), h_wide[s:e]) <= 1e-5
        assert max_rel_error(rd("dlam"), g[0][s:e]) <= 1e-5
        assert max_rel_error(rd("dx"), g[1][s:e]) <= 1e-5
        if r == 0:
            assert max_rel_error(np.fromfile(tmp_path / "out_0_dh0.bin", dtype=np.float32), g[2]) <= 1e-5
