"""CPU-side checks of the drop-in boundary (no compute calls without a GPU).

* liblinrec_cuda.so loads and exports every symbol include/linrec_cuda.h declares;
* the `linrec` module mirrors the reference module's surface and argument
  errors (proj/tests/python/test_smoke.py:87-115, linrec_py.cpp:21-89);
* without a CUDA device the product fails loudly -- there is no CPU path.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden


def test_library_exports_every_declared_symbol():
    from paper_1709_04057_b200 import capi
    declared = capi.declared_symbols()
    assert len(declared) >= 20
    lib = ctypes.CDLL(capi.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared) <= exported
    # nothing but the C ABI is exported
    assert all(s.startswith("linrec_") for s in exported), sorted(s for s in exported if not s.startswith("linrec_"))


def test_library_is_sm100a_only():
    from paper_1709_04057_b200 import capi
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    archs = {l.split(".")[-2] for l in out.splitlines() if l.strip().endswith(".cubin")}
    assert archs == {"sm_100a"}, archs


def test_abi_version_and_workspace_query():
    from paper_1709_04057_b200 import capi
    assert capi.lib.linrec_abi_version() == 1
    b = capi.lib.linrec_workspace_bytes(65536, 8192, 4)
    # control block + one flag and two carry records per tile, << the data (2 GiB/array)
    assert 0 < b < (1 << 30)
    assert capi.lib.linrec_workspace_bytes(0, 8, 4) == 0


def test_module_surface_matches_reference():
    from paper_1709_04057_b200 import linrec
    for name in ("scan", "scan_backward", "plan_chunks", "predicted_speedup", "hardware_workers"):
        assert hasattr(linrec, name)
    g = load_golden("frozen")
    assert linrec.plan_chunks(10, 4) == [tuple(r) for r in g["plan_10_4"].tolist()]
    assert linrec.plan_chunks(3, 8) == [(1, 1), (2, 2), (3, 3)]
    assert linrec.predicted_speedup(1, 1000) == pytest.approx(1 / 3)
    assert 0.95 <= linrec.predicted_speedup(3, 100000) <= 1.0
    assert linrec.predicted_speedup(8, 1 << 20) > 2.0
    assert linrec.hardware_workers() >= 1
    with pytest.raises(RuntimeError):
        linrec.plan_chunks(0, 4)
    with pytest.raises(RuntimeError):
        linrec.plan_chunks(4, 0)


def test_argument_errors_match_reference():
    """test_smoke.py:102-111 plus the messages of recurrence.hpp:39-51."""
    from paper_1709_04057_b200 import linrec
    ok = np.zeros((4, 1, 2))
    with pytest.raises(TypeError):
        linrec.scan(ok.astype(np.int64), ok.astype(np.int64))
    with pytest.raises(TypeError):
        linrec.scan(ok, ok.astype(np.float32))
    with pytest.raises(ValueError):
        linrec.scan(np.zeros((4, 2)), np.zeros((4, 2)))
    with pytest.raises(ValueError):
        linrec.scan(ok, ok, mode="speculative")
    with pytest.raises(ValueError):
        linrec.scan(ok, ok, workers=-1)
    with pytest.raises(RuntimeError, match=r"recurrence: shape mismatch, \[4,1,2\] vs \[4,1,3\]"):
        linrec.scan(ok, np.zeros((4, 1, 3)))
    with pytest.raises(RuntimeError, match=r"initial state \[1,3\] does not match \[1,2\]"):
        linrec.scan(ok, ok, np.zeros((1, 3)))
    with pytest.raises(RuntimeError, match="dimensions must be >= 1"):
        linrec.scan(np.zeros((0, 1, 2)), np.zeros((0, 1, 2)))
    with pytest.raises(RuntimeError, match=r"scan_backward\(h\): shape mismatch"):
        linrec.scan_backward(ok, None, np.zeros((3, 1, 2)), ok)
    with pytest.raises(TypeError):
        linrec.scan_backward(ok, None, ok.astype(np.float32), ok)


def test_no_cpu_fallback_without_gpu():
    from paper_1709_04057_b200 import capi, linrec
    if capi.lib.linrec_device_count() > 0:
        pytest.skip("a GPU is present")
    ok = np.zeros((4, 1, 2))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        linrec.scan(ok, ok)
    h = np.zeros_like(ok)
    rc = capi.lib.linrec_scan_host_f64(ok.ctypes.data, ok.ctypes.data, None, h.ctypes.data, 4, 2, 1, 0)
    assert rc == capi.ERR_CUDA


def test_import_fails_loudly_without_library(tmp_path):
    """Copy the package without its .so: importing must raise, not fall back."""
    import shutil
    pkg = os.path.join(ROOT, "paper_1709_04057_b200")
    dst = tmp_path / "paper_1709_04057_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    code = "import paper_1709_04057_b200"
    r = subprocess.run(["python", "-c", code], cwd=tmp_path, capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr


def test_product_does_not_import_oracle():
    """Only tests/, __graft_entry__.smoke() and bench.py may touch oracle/."""
    pkg = os.path.join(ROOT, "paper_1709_04057_b200")
    banned = ("import oracle", "from oracle", "liblinrec_oracle", "liblinrec_ref", "oracle/_ref")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not any(b in text for b in banned), f


def test_planner_kernel_counts():
    """linrec_scan_kernel_count (the planner, no GPU needed): one kernel for
    the per-channel, CTA-local and whole-chain cases; when the sequence is
    split into virtual segments, the scan + the fix-up + the decay-adaptive
    stitch's probe, reduce pass and carry fold (the unused ones exit at once,
    DESIGN.md 4)."""
    from paper_1709_04057_b200 import capi
    assert capi.scan_kernel_count(16, 1 << 20) == 1            # channels fill the GPU: per-channel kernel
    assert capi.scan_kernel_count(4096, 256) == 1              # C1: 43-tile chains stay whole
    assert capi.scan_kernel_count(4096, 256, backward=True) == 1
    assert capi.scan_kernel_count(1 << 20, 128) == 5           # C4: virtual segments + adaptive stitch
    assert capi.scan_kernel_count(1 << 20, 128, backward=True) == 5
    assert capi.scan_kernel_count(65536, 8192) == 4            # C2 forward: 4 segments, probe + unsplit twin
    assert capi.scan_kernel_count(65536, 8192, backward=True) == 1
    assert capi.scan_kernel_count(1 << 20, 128, mode=capi.SERIAL) == 1
    assert capi.scan_kernel_count(0, 128) == -1


def test_bench_host_inputs_shard_independent():
    """bench.py's host inputs: rows [r0, r1) generated alone equal the same
    rows of the global array, so the sequence-sharded ranks, the 1-GPU run,
    the CPU baseline and the reference arm all see one problem."""
    import numpy as np
    import bench
    full = bench.host_rows(1000, (2, 3), 0.05, 0.95, 7)
    assert full.dtype == np.float32 and full.shape == (1000, 2, 3)
    assert full.min() >= 0.05 and full.max() <= 0.95
    for world in (2, 3, 8):
        from paper_1709_04057_b200.sharded import segment_bounds
        parts = [bench.host_rows(1000, (2, 3), 0.05, 0.95, 7, *segment_bounds(1000, world, r))
                 for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)
    lam, x, h0, dh = bench.host_problem(64, 1, 4, 3)
    assert h0.shape == (1, 4) and lam.shape == x.shape == dh.shape == (64, 1, 4)


def test_column_blocks_partition_channels():
    """Channel sharding's column blocks (linrec_column_block, no GPU needed):
    contiguous, covering [0, W), multiples of 4 channels when W allows, longer
    first -- and the same as sharded.channel_shard."""
    from paper_1709_04057_b200 import capi, sharded
    for W in (1, 7, 128, 130, 8192, 65536):
        for n in (1, 2, 3, 8):
            blocks = [capi.column_block(W, n, d) for d in range(n)]
            assert blocks == [sharded.channel_shard(W, n, d) for d in range(n)]
            assert blocks[0][0] == 0 and blocks[-1][1] == W
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [e - s for s, e in blocks]
            assert sizes == sorted(sizes, reverse=True)
            if W % 4 == 0:
                assert all(s % 4 == 0 for s in sizes)
