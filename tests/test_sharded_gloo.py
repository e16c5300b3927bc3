"""Sequence / channel sharding orchestration on CPU: world_size 2 and 3 over
gloo (127.0.0.1), driving paper_1709_04057_b200.sharded with the reference
backend (tests/sharded_ref_backend.py), checked against the unsharded oracle
scan.  The CUDA kernels behind the same primitives are checked on the GPU in
tests/test_gpu_segments.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, T, b, n, rows, use_h0, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1709_04057_b200.sharded import SequenceShardedScan, segment_bounds
        from sharded_ref_backend import RefBackend
        rng = np.random.default_rng(seed)
        lam = rng.uniform(-1.0, 1.0, (T, b, n))
        x = rng.uniform(-1.0, 1.0, (T, b, n))
        h0 = rng.uniform(-1.0, 1.0, (b, n)) if use_h0 else None
        dh = rng.uniform(-1.0, 1.0, (T, b, n))
        s, e = segment_bounds(T, world, rank)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
        L, X, DH = t(lam[s:e]), t(x[s:e]), t(dh[s:e])
        H0 = t(h0) if use_h0 else None
        H = torch.empty_like(L)
        DL, DX = torch.empty_like(L), torch.empty_like(L)
        DH0 = torch.zeros(b, n, dtype=torch.float64)
        runner = SequenceShardedScan(T, b * n, backend=RefBackend(rows), device=torch.device("cpu"))
        # the runner allocates float32 scratch; the reference backend works in float64
        for name in ("seg_prod_f", "seg_prod_b", "agg", "aggs", "c_in", "y_in", "dh0_loc", "ones", "zeros"):
            setattr(runner, name, getattr(runner, name).double())
        runner.forward(L, X, H0, H)
        runner.backward(L, H0, H, DH, DL, DX, DH0)
        # a standalone backward with the halo exchange must agree too
        runner.hprev = None
        DL2, DX2 = torch.empty_like(L), torch.empty_like(L)
        DH02 = torch.zeros(b, n, dtype=torch.float64)
        runner.backward(L, H0, H, DH, DL2, DX2, DH02)
        q.put((rank, s, e, H.numpy(), DL.numpy(), DX.numpy(), DH0.numpy(), DL2.numpy(), DX2.numpy(), DH02.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,rows,use_h0", [(2, 23, 5, True), (3, 31, 4, False), (2, 8, 3, True), (3, 9, 2, True)])
def test_sequence_sharded_matches_unsharded(oracle, world, T, rows, use_h0):
    b, n, seed = 2, 3, 100 + world * T
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, b, n, rows, use_h0, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    lam = rng.uniform(-1.0, 1.0, (T, b, n))
    x = rng.uniform(-1.0, 1.0, (T, b, n))
    h0 = rng.uniform(-1.0, 1.0, (b, n)) if use_h0 else None
    dh = rng.uniform(-1.0, 1.0, (T, b, n))
    h_ref = oracle.scan_serial(lam, x, h0)
    dl_ref, dx_ref, dh0_ref = oracle.scan_backward(lam, h0, h_ref, dh)
    from oracle.oracle import max_rel_error
    for rank, s, e, H, DL, DX, DH0, DL2, DX2, DH02 in outs:
        assert max_rel_error(H, h_ref[s:e]) < 1e-12, rank
        for a, b_ in ((DL, dl_ref[s:e]), (DX, dx_ref[s:e]), (DL2, dl_ref[s:e]), (DX2, dx_ref[s:e])):
            assert max_rel_error(a, b_) < 1e-12, rank
        if rank == 0:
            assert max_rel_error(DH0, dh0_ref) < 1e-12
            assert max_rel_error(DH02, dh0_ref) < 1e-12


def test_segment_and_channel_bounds():
    from paper_1709_04057_b200.sharded import channel_shard, segment_bounds
    for T in (1, 7, 8, 1 << 20):
        for world in (1, 2, 3, 8):
            b = [segment_bounds(T, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == T
            assert all(e == s2 for (_, e), (s2, _) in zip(b, b[1:]))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert channel_shard(8192 * 8, 8, 3) == (3 * 8192, 4 * 8192)


def _channel_worker(rank, world, port, T, b, n, seed, q):
    """One rank of sharded.ChannelShardedScan with gather=True over gloo; the
    column entry points (linrec_scan_host_columns_*: CUDA) are replaced by the
    oracle on the rank's column block, so this checks the partition, the
    per-rank column writes and the host all-gather."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes
        from oracle.oracle import Oracle
        from paper_1709_04057_b200 import capi, sharded
        orc = Oracle()

        def arr(ptr, shape):
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)), shape)

        def cols_fwd(lam, x, h0, h, T_, W, c0, c1, mode, dtype_bytes, device):
            L, X, H = (arr(p, (T_, W)) for p in (lam, x, h))
            H0 = arr(h0, (W,))[None, c0:c1].copy() if h0 else None
            H[:, c0:c1] = orc.scan_serial(L[:, None, c0:c1].copy(), X[:, None, c0:c1].copy(),
                                          H0)[:, 0, :]

        def cols_bwd(lam, h0, h, dh, dlam, dx, dh0, T_, W, c0, c1, mode, dtype_bytes, device):
            L, H, DHh, DL, DX = (arr(p, (T_, W)) for p in (lam, h, dh, dlam, dx))
            D0 = arr(dh0, (W,))
            H0 = arr(h0, (W,))[None, c0:c1].copy() if h0 else None
            g = orc.scan_backward(L[:, None, c0:c1].copy(), H0, H[:, None, c0:c1].copy(),
                                  DHh[:, None, c0:c1].copy())
            DL[:, c0:c1], DX[:, c0:c1], D0[c0:c1] = g[0][:, 0], g[1][:, 0], g[2][0]

        capi.scan_host_columns = cols_fwd
        capi.scan_backward_host_columns = cols_bwd
        rng = np.random.default_rng(seed)
        lam = rng.uniform(0.05, 0.95, (T, b, n))
        x = rng.uniform(-1.0, 1.0, (T, b, n))
        h0 = rng.uniform(-1.0, 1.0, (b, n))
        dh = rng.uniform(-1.0, 1.0, (T, b, n))
        run = sharded.ChannelShardedScan(device=0)
        h = run.scan(lam, x, h0, gather=True)
        g = run.scan_backward(lam, h0, h, dh, gather=True)
        q.put((rank, run.columns(b * n), h, g[0], g[1], g[2]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,b,n", [(2, 40, 2, 8), (3, 17, 1, 13)])
def test_channel_sharded_scan_gather(oracle, world, T, b, n):
    seed = 7 + world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_channel_worker, args=(r, world, port, T, b, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(seed)
    lam = rng.uniform(0.05, 0.95, (T, b, n))
    x = rng.uniform(-1.0, 1.0, (T, b, n))
    h0 = rng.uniform(-1.0, 1.0, (b, n))
    dh = rng.uniform(-1.0, 1.0, (T, b, n))
    h_ref = oracle.scan_serial(lam, x, h0)
    g_ref = oracle.scan_backward(lam, h0, h_ref, dh)
    blocks = sorted(o[1] for o in outs)
    assert blocks[0][0] == 0 and blocks[-1][1] == b * n
    assert all(a[1] == c[0] for a, c in zip(blocks, blocks[1:]))
    for rank, cols, h, dl, dx, d0 in outs:  # every rank holds the full, gathered result
        assert np.array_equal(h, h_ref)
        for a, r in zip((dl, dx, d0), g_ref):
            assert np.array_equal(a, r)
