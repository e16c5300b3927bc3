"""Deep decoupled look-back (scan_chained.cuh::Lookback): with every tile of
a long sequence on ONE chain (LINREC_CHAINS=1, no virtual segments) a tile's
walk steps back over many published aggregates and applies them in batches
of four positions.  The chained scans must still match the bit-exact serial
kernel within the fp32 / fp64 bars and be bit-identical run to run (the
aggregates are applied oldest first whatever depth the walk reached).

LINREC_CHAINS is read once per process, so the checks run in a subprocess.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import torch
from paper_1709_04057_b200 import capi, torch_ops as ops
out = []
for policy in (capi.KERNEL_AUTO, capi.KERNEL_REGISTER):
    capi.set_kernel_policy(policy)
    for T, W, dt in ((1 << 18, 128, torch.float32), (1 << 16, 32, torch.float32),
                     (40000, 12, torch.float32), (1 << 16, 64, torch.float64)):
        g = torch.Generator(device="cuda").manual_seed(T + W)
        lam = torch.empty(T, 1, W, device="cuda", dtype=dt).uniform_(0.5, 1.0, generator=g)
        x = torch.empty_like(lam).uniform_(-1, 1, generator=g)
        dh = torch.empty_like(lam).uniform_(-1, 1, generator=g)
        h0 = torch.empty(1, W, device="cuda", dtype=dt).uniform_(-1, 1, generator=g)
        h = ops.scan(lam, x, h0)
        hs = ops.scan(lam, x, h0, mode="serial")
        same = bool(torch.equal(h, ops.scan(lam, x, h0)))
        gp = ops.scan_backward(lam, h0, hs, dh)
        gs = ops.scan_backward(lam, h0, hs, dh, mode="serial")
        same = same and all(torch.equal(a, b) for a, b in zip(gp, ops.scan_backward(lam, h0, hs, dh)))
        err = [((h - hs).abs().max() / hs.abs().max()).item()]
        err += [((a - b).abs().max() / b.abs().max()).item() for a, b in zip(gp, gs)]
        out.append({"policy": policy, "T": T, "W": W, "f64": dt == torch.float64,
                    "kernels": capi.scan_kernel_count(T, W, False, dtype_bytes=lam.element_size()),
                    "err": err, "same": same})
print(json.dumps(out))
"""


def test_single_chain_deep_lookback():
    env = dict(os.environ, LINREC_CHAINS="1")
    r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, timeout=600,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    cases = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(cases) == 8
    for c in cases:
        assert c["kernels"] == 1, c  # one chain per column: no stitch launch
        tol = 1e-12 if c["f64"] else 1e-5
        assert max(c["err"]) <= tol, c
        assert c["same"], c
