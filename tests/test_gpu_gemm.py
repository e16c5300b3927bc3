"""tcgen05 GEMM (csrc/gemm_tc.cuh) against an fp64 product, through the C ABI.

TF32 keeps 10 mantissa bits of the operands (fp32 accumulate): normwise error
bar 2e-3.  3xTF32 (LINREC_PREC_FP32, the layers' default) splits each operand
into hi + lo and must land at fp32-grade accuracy: 1e-5 normwise against the
exact product (an fp32 dot product of length K already carries ~K*2^-24)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {0: 1e-5, 1: 2e-3}  # PREC_FP32 (3xTF32), PREC_TF32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(M, N, K, a_mn, b_mn, accumulate=False, splits=1, seed=0, precision=0):
    from paper_1709_04057_b200 import capi
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.rand(M, K, device="cuda", generator=g) * 2 - 1
    B = torch.rand(N, K, device="cuda", generator=g) * 2 - 1
    C0 = torch.rand(M, N, device="cuda", generator=g) if accumulate else torch.zeros(M, N, device="cuda")
    Ast = A.t().contiguous() if a_mn else A
    Bst = B.t().contiguous() if b_mn else B
    ldc = (N + 3) // 4 * 4
    Cbuf = torch.zeros(M, ldc, device="cuda")
    Cbuf[:, :N] = C0
    scratch = torch.empty(capi.gemm_scratch_bytes(M, N, splits) // 4 + 1, device="cuda") if splits > 1 else None
    capi.gemm(Ast.data_ptr(), a_mn, Ast.shape[1], Bst.data_ptr(), b_mn, Bst.shape[1], Cbuf.data_ptr(), ldc, M, N,
              K, accumulate, precision, splits, None if scratch is None else scratch.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t() + (C0.double() if accumulate else 0)
    return ((Cbuf[:, :N].double() - ref).abs().max() / ref.abs().max()).item()


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (256, 256, 512), (300, 200, 100), (1000, 384, 1024)])
def test_gemm_layouts(a_mn, b_mn, M, N, K, precision):
    assert run(M, N, K, a_mn, b_mn, precision=precision) < TOL[precision]


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("splits", [2, 7, 16])
def test_gemm_split_k_and_accumulate(splits, precision):
    assert run(512, 256, 4096, True, True, accumulate=True, splits=splits, precision=precision) < TOL[precision]
    assert run(256, 512, 2048, False, True, accumulate=True, splits=1, precision=precision) < TOL[precision]


def test_gemm_many_tiles_persistent():
    # more tiles than CTA pairs: every pair walks several tiles through both TMEM accumulators
    assert run(8192, 1024, 256, False, False) < TOL[0]
    assert run(20000, 640, 96, False, True, precision=1) < TOL[1]
    assert run(300, 1000, 4096, True, False, splits=5) < TOL[0]


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("N", [1, 3, 4, 8])
def test_gemm_skinny_cuda_core_path(N, precision):
    # <= 8 output columns: exact fp32 FMAs on CUDA cores (gemm_tc.cu::gemm_skinny), fp32-grade in both modes
    bmn = N % 4 == 0  # an MN-major B needs a 16-byte pitch (the ABI's TMA rule)
    assert run(5000, N, 512, False, bmn, precision=precision) < 1e-5      # dx = dpre . W (rows kernel)
    assert run(777, N, 100, False, False, accumulate=True) < 1e-5
    assert run(1001, N, 516, False, bmn) < 1e-5
    assert run(512, N, 65536, True, bmn, splits=16, precision=precision) < 1e-5  # weight gradient (split-K)
    assert run(300, N, 3000, True, False, accumulate=True, splits=5) < 1e-5
    assert run(300, N, 3000, True, bmn, splits=1) < TOL[0]               # no scratch: tensor cores


def test_tf32_operand_truncation():
    """The tensor core reads tf32 by dropping the low 13 mantissa bits; the
    3xTF32 split (lo = v - trunc(v)) relies on it.  A one-hot B picks single
    operands out so the MMA's view of them is visible."""
    from paper_1709_04057_b200 import capi
    M, N, K = 128, 32, 32
    base = torch.tensor([1.0 + 2.0 ** -12 * k for k in range(M)], device="cuda")  # sub-tf32 bits
    A = torch.zeros(M, K, device="cuda")
    A[:, 0] = base
    B = torch.zeros(N, K, device="cuda")
    B[0, 0] = 1.0
    C = torch.zeros(M, N, device="cuda")
    capi.gemm(A.data_ptr(), False, K, B.data_ptr(), False, K, C.data_ptr(), N, M, N, K, False, capi.PREC_TF32, 1,
              None, torch.cuda.current_stream().cuda_stream)
    C3 = torch.zeros(M, N, device="cuda")
    capi.gemm(A.data_ptr(), False, K, B.data_ptr(), False, K, C3.data_ptr(), N, M, N, K, False, capi.PREC_FP32, 1,
              None, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    trunc = (base.view(torch.int32) & ~0x1FFF).view(torch.float32)
    assert torch.equal(C[:, 0], trunc)
    assert torch.equal(C3[:, 0], base)  # 3xTF32 recovers the operand exactly


def test_gemm_deterministic():
    from paper_1709_04057_b200 import capi
    M, N, K = 2048, 512, 8192
    A = torch.rand(K, M, device="cuda")
    B = torch.rand(K, N, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.zeros(M, N, device="cuda")
        scratch = torch.empty(capi.gemm_scratch_bytes(M, N, 16) // 4, device="cuda")
        capi.gemm(A.data_ptr(), True, M, B.data_ptr(), True, N, C.data_ptr(), N, M, N, K, False, capi.PREC_FP32, 16,
                  scratch.data_ptr(), torch.cuda.current_stream().cuda_stream)
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


def test_gemm_errors():
    from paper_1709_04057_b200 import capi
    A = torch.zeros(8, 8, device="cuda")
    with pytest.raises(capi.LinrecError, match="precision"):
        capi.gemm(A.data_ptr(), False, 8, A.data_ptr(), False, 8, A.data_ptr(), 8, 8, 8, 8, precision=7)
    with pytest.raises(capi.LinrecError, match="16-byte"):
        capi.gemm(A.data_ptr(), False, 7, A.data_ptr(), False, 8, A.data_ptr(), 8, 8, 8, 7)
