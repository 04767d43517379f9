"""Kernel time breakdown of the GPU front end (torch.profiler / CUPTI)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2101_05063_b200.hessenberg import hessenberg_device  # noqa: E402

n = int(sys.argv[1])
A0 = torch.randn((n, n), dtype=torch.float64, device="cuda")
A = A0.clone()
hessenberg_device(A)
A = A0.clone()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    hessenberg_device(A)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
