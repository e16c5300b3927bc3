"""Developer probe: one bench_model step (parallel) between cudaProfilerStart
and Stop, for `ncu --profile-from-start off` launch lists.
Usage: bm_profile.py ARCH T [precision]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from bench_model import Model  # noqa: E402

arch, T = sys.argv[1], int(sys.argv[2])
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
b = 65536 // T
gen = torch.Generator().manual_seed(1)
model = Model(arch, 4, 256, gen, prec)
dev = torch.device("cuda", 0)
x = (torch.rand(T, b, 4, generator=gen) * 2 - 1).to(dev)
zero = torch.zeros(b, 256, device=dev)
for _ in range(3):
    model.step(x, zero, "parallel")
torch.cuda.synchronize()
torch.cuda.profiler.start()
model.step(x, zero, "parallel")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
