"""GPU check of the sequence-sharding kernels (segment scans, carry folding,
fix-ups): R ranks are emulated in one process on one GPU -- the all-gather is
a copy -- and the stitched result is compared with the oracle's unsharded
scan.  The orchestration itself (SequenceShardedScan over a process group) is
covered on CPU by tests/test_sharded_gloo.py and, with NCCL, by the world-1
case below."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    from oracle.oracle import max_rel_error
    return max_rel_error(a, b)


def emulate(lam, x, h0, dh, R):
    """Run the per-rank segment protocol for R ranks sequentially."""
    from paper_1709_04057_b200 import capi
    from paper_1709_04057_b200.sharded import segment_bounds
    T, W = lam.shape
    es = lam.element_size()  # 4: fp32, 8: fp64
    st = torch.cuda.current_stream().cuda_stream
    dev = lam.device
    h = torch.empty_like(lam)
    dlam, dx = torch.empty_like(lam), torch.empty_like(lam)
    dh0 = torch.empty(W, device=dev, dtype=lam.dtype)
    aggs = torch.zeros(R, 2, W, device=dev, dtype=lam.dtype)
    segs, sp_f, sp_b, rows_f, rows_b = [], [], [], [], []
    for r in range(R):
        s, e = segment_bounds(T, R, r)
        segs.append((s, e))
        rf, rb = capi.segment_tile_rows(e - s, W, False, es), capi.segment_tile_rows(e - s, W, True, es)
        rows_f.append(rf)
        rows_b.append(rb)
        sp_f.append(torch.empty(capi.segment_prod_rows(e - s, W, False, es), W, device=dev, dtype=lam.dtype))
        sp_b.append(torch.empty(capi.segment_prod_rows(e - s, W, True, es), W, device=dev, dtype=lam.dtype))
    # forward: local scans
    for r, (s, e) in enumerate(segs):
        capi.segment_scan(lam[s].data_ptr(), x[s].data_ptr(), h0.data_ptr() if r == 0 else None, h[s].data_ptr(),
                          sp_f[r].data_ptr(), aggs[r].data_ptr(), e - s, W, es, None, st)
    aggs[0, 0].zero_()
    c_in = [h0] + [torch.empty(W, device=dev, dtype=lam.dtype) for _ in range(1, R)]
    for r in range(R):  # every rank: the fix-up also stitches its own virtual segments
        s, e = segs[r]
        if r > 0:
            capi.compose_carries(aggs.data_ptr(), 0, r, 1, None, c_in[r].data_ptr(), W, es, st)
        capi.segment_fixup(lam[s].data_ptr(), h[s].data_ptr(), sp_f[r].data_ptr(),
                           c_in[r].data_ptr() if r > 0 else None, e - s, W, rows_f[r], es, st)
    # backward
    ones = torch.ones(W, device=dev, dtype=lam.dtype)
    dh0_loc = [torch.empty(W, device=dev, dtype=lam.dtype) for _ in range(R)]
    baggs = torch.zeros(R, 2, W, device=dev, dtype=lam.dtype)
    for r, (s, e) in enumerate(segs):
        ln = ones if r < R - 1 else None
        capi.segment_scan_backward(lam[s].data_ptr(), c_in[r].data_ptr(), h[s].data_ptr(), dh[s].data_ptr(),
                                   None if ln is None else ln.data_ptr(), dlam[s].data_ptr(), dx[s].data_ptr(),
                                   dh0_loc[r].data_ptr(), sp_b[r].data_ptr(), baggs[r].data_ptr(), e - s, W, es,
                                   None, st)
    y0 = torch.zeros(W, device=dev, dtype=lam.dtype)
    for r, (s, e) in enumerate(segs):
        y = None
        if r < R - 1:
            y = torch.empty(W, device=dev, dtype=lam.dtype)
            capi.compose_carries(baggs.data_ptr(), R - 1, r, -1, None, y.data_ptr(), W, es, st)
            if r == 0:
                y0 = y
        ln = ones if r < R - 1 else None
        capi.segment_fixup_backward(lam[s].data_ptr(), c_in[r].data_ptr(), h[s].data_ptr(),
                                    None if ln is None else ln.data_ptr(), sp_b[r].data_ptr(),
                                    None if y is None else y.data_ptr(), dlam[s].data_ptr(), dx[s].data_ptr(), e - s,
                                    W, rows_b[r], es, st)
    capi.compose_carries(baggs.data_ptr(), 0, 1, 1, y0.data_ptr(), dh0.data_ptr(), W, es, st)
    torch.cuda.synchronize()
    return h, dlam, dx, dh0


@pytest.mark.parametrize("T,W,lo,hi,R", [
    (65536, 128, 0.05, 0.95, 4),    # the 1M-step regime, scaled: underflow after ~100 rows
    (65536, 128, 0.05, 0.95, 8),
    (20000, 40, 0.999, 1.0, 3),     # decays ~1: the fix-up covers whole segments
    (5000, 256, -1.0, 1.0, 2),
    (3001, 7, 0.05, 0.95, 5),       # W % 4 != 0: register kernels, scalar fix-up
    (700, 16, 0.9, 1.0, 8),
    (9000, 512, 0.05, 0.95, 3),     # W > 256: the rank aggregate from the fold kernel
])
def test_emulated_sequence_sharding(oracle, T, W, lo, hi, R):
    rng = np.random.default_rng(T + W + R)
    lam = rng.uniform(lo, hi, (T, W)).astype(np.float32)
    x = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (W,)).astype(np.float32)
    dh = rng.uniform(-1, 1, (T, W)).astype(np.float32)
    cu = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    h, dlam, dx, dh0 = emulate(cu(lam), cu(x), cu(h0), cu(dh), R)
    ref = oracle.scan_serial(lam, x, h0)
    assert rel(h.cpu().numpy(), ref) <= 1e-5
    wide = oracle.scan_serial_wide(lam, x, h0)
    assert rel(h.cpu().numpy(), wide) <= 1e-5
    g = oracle.scan_backward_wide(lam, h0, ref, dh)
    for a, r in zip((dlam, dx, dh0), g):
        assert rel(a.cpu().numpy(), r) <= 1e-5


@pytest.mark.parametrize("T,W,lo,hi,R", [(65536, 128, 0.05, 0.95, 4), (3001, 7, 0.05, 0.95, 5),
                                         (9000, 512, 0.05, 0.95, 3)])
def test_emulated_sequence_sharding_fp64(oracle, T, W, lo, hi, R):
    """fp64 segments: the fold kernel (no tail fold in double) and the fix-up's
    carry fold in double; 1e-12 normwise against the unsharded serial scan."""
    rng = np.random.default_rng(T + W + R + 1)
    lam = rng.uniform(lo, hi, (T, W))
    x = rng.uniform(-1, 1, (T, W))
    h0 = rng.uniform(-1, 1, (W,))
    dh = rng.uniform(-1, 1, (T, W))
    cu = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    h, dlam, dx, dh0 = emulate(cu(lam), cu(x), cu(h0), cu(dh), R)
    ref = oracle.scan_serial(lam, x, h0)
    assert rel(h.cpu().numpy(), ref) <= 1e-12
    g = oracle.scan_backward(lam, h0, ref, dh)
    for a, r in zip((dlam, dx, dh0), g):
        assert rel(a.cpu().numpy(), r) <= 1e-12


def test_runner_world_one_nccl(oracle):
    """SequenceShardedScan with the CUDA backend over a 1-rank NCCL group."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1709_04057_b200.sharded import SequenceShardedScan
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        T, b, n = 30000, 1, 128
        rng = np.random.default_rng(1)
        lam = rng.uniform(0.05, 0.95, (T, b, n)).astype(np.float32)
        x = rng.uniform(-1, 1, (T, b, n)).astype(np.float32)
        h0 = rng.uniform(-1, 1, (b, n)).astype(np.float32)
        dh = rng.uniform(-1, 1, (T, b, n)).astype(np.float32)
        cu = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        L, X, H0, DH = cu(lam), cu(x), cu(h0), cu(dh)
        H = torch.empty_like(L)
        DL, DX, DH0 = torch.empty_like(L), torch.empty_like(L), torch.empty_like(H0)
        run = SequenceShardedScan(T, b * n)
        run.forward(L, X, H0, H)
        run.backward(L, H0, H, DH, DL, DX, DH0)
        torch.cuda.synchronize()
        ref = oracle.scan_serial(lam, x, h0)
        assert rel(H.cpu().numpy(), ref) <= 1e-5
        for a, r in zip((DL, DX, DH0), oracle.scan_backward(lam, h0, ref, dh)):
            assert rel(a.cpu().numpy(), r) <= 1e-5
    finally:
        dist.destroy_process_group()
