"""The reference's property suite (proj/include/linrec/verify.hpp:178-294) run
against the GPU path: serial-vs-parallel equivalence over 200 random
instances, the closed-form identities, exact two-segment composition, the
recurrence backward against central finite differences -- and the suite's
own test-of-the-test (verify.hpp:285-286: a flipped d_decays must fail the
finite-difference check).  Serial is the per-channel kernel (bit-exact to the
reference's scan_serial); parallel is whatever kernel family the dispatch
picks (cluster, CTA-local, TMA chained with virtual segments and the
decay-adaptive stitch), so the sweep also runs through every family.

Metric as verify.hpp:49-56: max|a - b| / max|serial|."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _p(t):
    return None if t is None else t.data_ptr()


def _scan(lam, x, h0, mode):
    from paper_1709_04057_b200 import capi
    T, W = lam.shape
    h = torch.empty_like(lam)
    capi.scan(_p(lam), _p(x), _p(h0), _p(h), T, W, mode, lam.element_size())
    return h


def _backward(lam, h0, h, dh, mode):
    from paper_1709_04057_b200 import capi
    T, W = lam.shape
    dl, dx, d0 = torch.empty_like(lam), torch.empty_like(lam), torch.empty(W, dtype=lam.dtype, device="cuda")
    capi.scan_backward(_p(lam), _p(h0), _p(h), _p(dh), _p(dl), _p(dx), _p(d0), T, W, mode, lam.element_size())
    return dl, dx, d0


def _max_rel(a, ref):
    return ((a.double() - ref.double()).abs().max() / ref.double().abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.float64, 1e-10)])
def test_serial_vs_parallel_200_instances(dtype, tol):
    """verify.hpp:178-205: T in [1, 64], b = 2, n in {1, 3, 32}, every input
    ~ U(-1, 1); here 200 such instances plus every tenth one stretched to a
    long sequence, so the parallel side covers each kernel family."""
    from paper_1709_04057_b200 import capi
    rng = np.random.default_rng(1 if dtype == torch.float32 else 2)
    worst = 0.0
    families = set()
    for trial in range(200):
        T = int(1 + rng.integers(64))
        n = int(rng.choice([1, 3, 32]))
        if trial % 10 == 9:
            T = int(rng.choice([700, 4096, 30000]))
        W = 2 * n
        lam, x = (torch.from_numpy(rng.uniform(-1, 1, (T, W))).to("cuda", dtype) for _ in range(2))
        h0 = torch.from_numpy(rng.uniform(-1, 1, W)).to("cuda", dtype)
        dh = torch.from_numpy(rng.uniform(-1, 1, (T, W))).to("cuda", dtype)
        hs, hp = _scan(lam, x, h0, capi.SERIAL), _scan(lam, x, h0, capi.PARALLEL)
        gs = _backward(lam, h0, hs, dh, capi.SERIAL)
        gp = _backward(lam, h0, hs, dh, capi.PARALLEL)
        families.add(capi.scan_kernel_name(T, W, dtype_bytes=lam.element_size()))
        worst = max(worst, _max_rel(hp, hs), *(_max_rel(a, b) for a, b in zip(gp, gs)))
    torch.cuda.synchronize()
    assert worst <= tol, worst
    assert len(families) >= 2, families


@pytest.mark.parametrize("T", [33, 4096, 30000])
@pytest.mark.parametrize("mode_name", ["serial", "parallel"])
def test_identities_exact(T, mode_name):
    """verify.hpp:207-232: decay 1 gives exact prefix sums of integer
    impulses from an integer initial state, decay 0 passes the impulses
    through -- in every kernel family (T = 33 CTA-local, 4096 cluster, 30000
    chained with virtual segments; b = 2, n = 3 and a wide case)."""
    from paper_1709_04057_b200 import capi
    mode = capi.SERIAL if mode_name == "serial" else capi.PARALLEL
    rng = np.random.default_rng(T)
    for W in (6, 256):
        x = torch.from_numpy(rng.integers(-4, 5, (T, W)).astype(np.float64)).cuda()
        h0 = torch.from_numpy(rng.integers(-4, 5, W).astype(np.float64)).cuda()
        ones, zeros = torch.ones_like(x), torch.zeros_like(x)
        cum = _scan(ones, x, h0, mode)
        assert torch.equal(cum, h0 + torch.cumsum(x, 0))
        assert torch.equal(_scan(zeros, x, h0, mode), x)
        # fp32: the same sums are exact while they stay integers below 2^24
        x32, h032 = x.float(), h0.float()
        assert torch.equal(_scan(ones.float(), x32, h032, mode), (h0 + torch.cumsum(x, 0)).float())
        assert torch.equal(_scan(zeros.float(), x32, h032, mode), x32)


@pytest.mark.parametrize("T,cut", [(24, 11), (30000, 12345), (4096, 2048)])
def test_two_segment_composition(T, cut):
    """verify.hpp:234-265: scanning [0, cut) and restarting [cut, T) from the
    state at cut - 1 reproduces the full scan -- exactly in serial mode,
    within the fp64 tolerance in parallel mode."""
    from paper_1709_04057_b200 import capi
    rng = np.random.default_rng(T + cut)
    W = 8
    lam, x = (torch.from_numpy(rng.uniform(-1, 1, (T, W))).cuda() for _ in range(2))
    h0 = torch.from_numpy(rng.uniform(-1, 1, W)).cuda()
    for mode in (capi.SERIAL, capi.PARALLEL):
        full = _scan(lam, x, h0, mode)
        head = _scan(lam[:cut].contiguous(), x[:cut].contiguous(), h0, mode)
        tail = _scan(lam[cut:].contiguous(), x[cut:].contiguous(), head[-1].contiguous(), mode)
        both = torch.cat([head, tail])
        if mode == capi.SERIAL:
            assert torch.equal(both, full)
        else:
            assert _max_rel(both, full) <= 1e-10


def _fd_worst(lam, x, h0, dh, grads):
    """verify.hpp:69-118: central differences (eps 1e-6) of sum(h * dh) w.r.t.
    every decay, impulse and initial value, against the analytic gradients;
    relative gap where the scale exceeds 1e-7.  The forward is the GPU serial
    scan in fp64."""
    from paper_1709_04057_b200 import capi

    def loss(l_, x_, h0_):
        return float((_scan(l_, x_, h0_, capi.SERIAL) * dh).sum().item())

    worst = 0.0
    for which, g in zip(range(3), grads):
        base = [lam.clone(), x.clone(), h0.clone()]
        flat = base[which].view(-1)
        gflat = g.reshape(-1)
        for i in range(flat.numel()):
            saved = flat[i].item()
            flat[i] = saved + 1e-6
            up = loss(*base)
            flat[i] = saved - 1e-6
            down = loss(*base)
            flat[i] = saved
            numeric = (up - down) / 2e-6
            analytic = gflat[i].item()
            scale = max(abs(numeric), abs(analytic))
            if scale > 1e-7:
                worst = max(worst, abs(numeric - analytic) / scale)
    return worst


@pytest.mark.parametrize("mode_name", ["serial", "parallel"])
def test_backward_finite_differences(mode_name):
    """verify.hpp:267-294 (T = 7, b = 2, n = 3, fp64): the GPU backward
    (d_decays, d_impulses, d_initial) agrees with central differences
    within 1e-5 -- and flipping d_decays, the suite's injected fault
    (verify.hpp:285-286), must break that agreement."""
    from paper_1709_04057_b200 import capi
    mode = capi.SERIAL if mode_name == "serial" else capi.PARALLEL
    rng = np.random.default_rng(4)
    T, W = 7, 6
    lam, x, dh = (torch.from_numpy(rng.uniform(-1, 1, (T, W))).cuda() for _ in range(3))
    h0 = torch.from_numpy(rng.uniform(-1, 1, W)).cuda()
    h = _scan(lam, x, h0, capi.SERIAL)
    dl, dx, d0 = _backward(lam, h0, h, dh, mode)
    assert _fd_worst(lam, x, h0, dh, (dl, dx, d0)) <= 1e-5
    assert _fd_worst(lam, x, h0, dh, (-dl, dx, d0)) > 1e-5  # the test of the test


def test_workers_do_not_change_results():
    """verify.hpp:474-506 (worker invariance) and test_recurrence.cpp:173-183
    (bit-determinism for a plan): the Python module's `workers` argument is
    validated but does not shape the GPU plan, so results are bit-identical
    across worker counts and runs."""
    from paper_1709_04057_b200 import linrec
    rng = np.random.default_rng(257)
    lam = rng.uniform(-1, 1, (257, 2, 3)).astype(np.float32)
    x = rng.uniform(-1, 1, (257, 2, 3)).astype(np.float32)
    h0 = rng.uniform(-1, 1, (2, 3)).astype(np.float32)
    outs = [linrec.scan(lam, x, h0, workers=w) for w in (0, 2, 3, 8, 16, 2)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
