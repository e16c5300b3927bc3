import json,sys
for f in sys.argv[1:]:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, "ms/step", round(d["ms_per_step"],3), "value", "%.3e"%d["value"], "gemm_tflops", round(d["gemm_tflops_total"],1), "gemm_share", round(d["gemm_share_of_step"],3))
    for k,v in d["stages"].items(): print("   ",k, {a:round(b,3) for a,b in v.items()})
