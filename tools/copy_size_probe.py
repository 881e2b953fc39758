"""Plain device-to-device copy (torch dst.copy_(src), contiguous) at several sizes: the
achievable HBM copy rate as a function of traffic per launch -- the denominator the
mid-size fractions should be read against (MEASURED_PEAKS.json is a 2 GiB copy).  Also
cudaMemcpyAsync D2D through torch (same thing) -- CUDA-graph timed, median of 3."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from timing import t
out = {}
for mib in (16, 36, 72, 144, 288, 576, 1152):
    n = mib << 20
    a = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    us = t(lambda: b.copy_(a), it=10)
    out[f"{mib}MiB"] = [round(us, 2), round(2 * n / us / 1e3, 1)]
    del a, b
print(json.dumps({"copy_MiB: [us, GB/s read+write]": out}))
