import sys, os, re
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1709_04057_b200 import capi
T, W = 65536, 8192
lam = torch.rand(T, W, device="cuda") * 0.9 + 0.05
x = torch.rand(T, W, device="cuda")
h = torch.empty_like(lam)
st = torch.cuda.current_stream().cuda_stream
f = lambda: capi.scan(lam.data_ptr(), x.data_ptr(), None, h.data_ptr(), T, W, capi.PARALLEL, 4, None, st)
f(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    f(); f(); torch.cuda.synchronize()
OUR = re.compile(r"linrec_|\btc::|\blayers::|\btrain::")
names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
print(len(names), sum(1 for n in names if OUR.search(n)), names[:8])
print("kernel_count", capi.scan_kernel_count(T, W, False))
