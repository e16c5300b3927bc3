"""Channel sharding of HOST arrays (include/linrec_cuda.h
"channel sharding"): the columns of a [T][W] problem split over devices, each
block staged with 2-D copies -- no communication, because channels are
independent (recurrence.hpp:109).  On the one-GPU test box the "devices" are
device 0 repeated (one host thread per block), which exercises the column
staging, the per-thread pipelines and the reassembly exactly as N GPUs would.

Bars: mode "serial" bit-exact against the oracle's serial scan (and the
reference's golden fixtures); mode "parallel" <= 1e-5 normwise (fp32) /
1e-12 (fp64) like test_gpu_parity.py."""
import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.fixture(scope="module")
def sh():
    from paper_1709_04057_b200 import sharded
    return sharded


def rel(a, b):
    from oracle.oracle import max_rel_error
    return max_rel_error(a, b)


@pytest.mark.parametrize("T,b,n,ndev", [(1, 1, 1, 2), (300, 1, 130, 3), (1000, 3, 7, 2), (4096, 2, 256, 4),
                                        (70000, 1, 64, 2)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_matches_single_gpu_oracle(sh, oracle, T, b, n, ndev, dtype):
    lam, x, h0 = (a.astype(dtype) for a in oracle.random_recurrence(7, T, b, n, split=1000))
    dh = oracle.rng_fill(oracle.rng(8), (T, b, n), -1.0, 1.0).astype(dtype)
    devs = [0] * ndev
    h_ref = oracle.scan_serial(lam, x, h0)
    g_ref = oracle.scan_backward(lam, h0, h_ref, dh)
    hs = sh.channel_sharded_scan(lam, x, h0, devices=devs, mode="serial")
    assert np.array_equal(hs, h_ref)
    gs = sh.channel_sharded_scan_backward(lam, h0, hs, dh, devices=devs, mode="serial")
    assert all(np.array_equal(a, r) for a, r in zip(gs, g_ref))
    tol = 1e-5 if dtype == np.float32 else 1e-12
    hp = sh.channel_sharded_scan(lam, x, h0, devices=devs)
    assert rel(hp, h_ref) <= tol
    gp = sh.channel_sharded_scan_backward(lam, h0, h_ref, dh, devices=devs)
    assert max(rel(a, r) for a, r in zip(gp, g_ref)) <= tol


@pytest.mark.parametrize("name", ["t513_b2_n64_f32", "t129_b2_n66_f64", "t1000_b3_n7_f32"])
def test_golden_fixtures(sh, name):
    g = load_golden(name)
    hs = sh.channel_sharded_scan(g["lam"], g["x"], g["h0"], devices=[0, 0, 0], mode="serial")
    assert np.array_equal(hs, g["h_serial"])


def test_pinned_and_column_api(sh, oracle):
    """The C ABI column entry point on page-locked buffers (2-D DMA straight
    from / into the caller's strided block) writes exactly its columns."""
    from paper_1709_04057_b200 import capi
    T, b, n = 3000, 2, 96
    W = b * n
    lam, x, h0 = oracle.random_recurrence(3, T, b, n, split=1000)
    pin = [torch.from_numpy(a).pin_memory() for a in (lam, x, h0)]
    h = torch.full((T, b, n), -7.0).pin_memory()
    c0, c1 = 40, 132
    capi.scan_host_columns(pin[0].data_ptr(), pin[1].data_ptr(), pin[2].data_ptr(), h.data_ptr(), T, W, c0, c1,
                           capi.SERIAL, 4, 0)
    hn = h.numpy().reshape(T, W)
    ref = oracle.scan_serial(lam, x, h0).reshape(T, W)
    assert np.array_equal(hn[:, c0:c1], ref[:, c0:c1])
    assert np.all(hn[:, :c0] == -7.0) and np.all(hn[:, c1:] == -7.0)


def test_errors(sh, oracle):
    from paper_1709_04057_b200 import capi
    lam, x, h0 = oracle.random_recurrence(1, 10, 1, 8, split=1000)
    with pytest.raises(RuntimeError, match=r"recurrence: shape mismatch"):
        sh.channel_sharded_scan(lam, x[:-1], h0, devices=[0])
    with pytest.raises(TypeError):
        sh.channel_sharded_scan(lam, x.astype(np.float64), h0, devices=[0])
    with pytest.raises(capi.LinrecError, match="devices"):
        sh.channel_sharded_scan(lam, x, h0, devices=[99])
    with pytest.raises(capi.LinrecError, match="columns"):
        h = np.empty_like(lam)
        capi.scan_host_columns(lam.ctypes.data, x.ctypes.data, None, h.ctypes.data, 10, 8, 5, 3, capi.PARALLEL, 4, 0)
