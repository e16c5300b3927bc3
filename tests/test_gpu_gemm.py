"""tcgen05 TF32 GEMM (csrc/gemm_tc.cuh) against an fp64 product.

TF32 keeps 10 mantissa bits of the operands (fp32 accumulate), so the bar is
a normwise error of 2e-3 against the exact product -- the layer tolerance
declared in DESIGN.md follows from it."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(M, N, K, a_mn, b_mn, accumulate=False, splits=1, seed=0):
    from paper_1709_04057_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C0 = torch.rand(M, N, device="cuda", generator=g) if accumulate else torch.zeros(M, N, device="cuda")
    Ast = A.t().contiguous() if a_mn else A
    Bst = B.t().contiguous() if b_mn else B
    C = C0.clone()
    scratch = torch.empty(max(1, splits) * M * N, device="cuda") if splits > 1 else None
    capi.gemm_tf32(Ast.data_ptr(), a_mn, Ast.shape[1], Bst.data_ptr(), b_mn, Bst.shape[1], C.data_ptr(), N, M, N, K,
                   accumulate, splits, None if scratch is None else scratch.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t() + (C0.double() if accumulate else 0)
    return ((C.double() - ref).abs().max() / ref.abs().max()).item()


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 256, 512), (300, 200, 100), (1000, 384, 1024)])
def test_gemm_layouts(a_mn, b_mn, M, N, K):
    assert run(M, N, K, a_mn, b_mn) < 2e-3


@pytest.mark.parametrize("splits", [2, 7, 16])
def test_gemm_split_k_and_accumulate(splits):
    assert run(512, 256, 4096, True, True, accumulate=True, splits=splits) < 2e-3
    assert run(256, 512, 2048, False, True, accumulate=True, splits=1) < 2e-3


def test_gemm_deterministic():
    from paper_1709_04057_b200 import capi
    M, N, K = 2048, 512, 8192
    A = torch.rand(K, M, device="cuda")
    B = torch.rand(K, N, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.zeros(M, N, device="cuda")
        scratch = torch.empty(16 * M * N, device="cuda")
        capi.gemm_tf32(A.data_ptr(), True, M, B.data_ptr(), True, N, C.data_ptr(), N, M, N, K, False, 16,
                       scratch.data_ptr(), torch.cuda.current_stream().cuda_stream)
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
