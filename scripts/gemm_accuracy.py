"""Probe: normwise error of the tcgen05 GEMM vs K, precision and split-K,
against an fp64 product, with torch's fp32 SGEMM (no TF32) as a yardstick."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1709_04057_b200 import capi

torch.backends.cuda.matmul.allow_tf32 = False
st = torch.cuda.current_stream().cuda_stream
for K in (256, 1024, 4096, 16384, 65536, 262144):
    M, N = 512, 256
    A = torch.rand(K, M, device="cuda") * 2 - 1
    B = torch.rand(K, N, device="cuda") * 2 - 1
    ref = A.double().t() @ B.double()
    den = ref.abs().max().item()
    row = [f"K={K:7d}"]
    t = (A.t() @ B)
    row.append(f"torch_fp32={((t.double()-ref).abs().max().item()/den):.2e}")
    for prec in (0, 1):
        for splits in (1, 8, 64):
            if splits > K // 128:
                continue
            C = torch.zeros(M, N, device="cuda")
            scr = torch.empty(max(1, capi.gemm_scratch_bytes(M, N, splits) // 4), device="cuda")
            capi.gemm(A.data_ptr(), True, M, B.data_ptr(), True, N, C.data_ptr(), N, M, N, K, False, prec, splits,
                      scr.data_ptr(), st)
            torch.cuda.synchronize()
            row.append(f"{'3x' if prec == 0 else 'tf'}/s{splits}={((C.double()-ref).abs().max().item()/den):.2e}")
    print(" ".join(row), flush=True)
