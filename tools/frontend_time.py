"""Time the GPU front end (hsrq_hessenberg_reduce with Q, hsrq_backmultiply)
at size n and check the SPEC backward-error bounds.  python tools/frontend_time.py n"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_05063_b200.hessenberg import backmultiply_device, hessenberg_device  # noqa: E402

n = int(sys.argv[1])
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
for rep in range(2):
    A = A0.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Q = hessenberg_device(A)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
Am, Hm, Qm = A0.T, A.T, Q.T
eps = np.finfo(float).eps
orth = torch.linalg.norm(Qm.T @ Qm - torch.eye(n, dtype=torch.float64, device="cuda")).item()
sim = torch.linalg.norm(Qm.T @ Am @ Qm - Hm).item() / torch.linalg.norm(Am).item()
below = torch.count_nonzero(torch.tril(Hm, -2)).item()
flops = 10.0 / 3.0 * n ** 3 + 4.0 / 3.0 * n ** 3  # DGEHRD + DORGHR model
X = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=g)
torch.cuda.synchronize()
t0 = time.perf_counter()
Z = backmultiply_device(Q, X)
torch.cuda.synchronize()
tb = time.perf_counter() - t0
print(f"n={n}: reduce+Q {dt * 1e3:.1f} ms ({flops / dt / 1e12:.2f} TFLOP/s model), "
      f"||Q'Q-I||/(n eps)={orth / n / eps:.3f}  ||Q'AQ-H||/(n eps ||A||)={sim / n / eps:.3f}  "
      f"nonzeros below subdiag={below}; back-multiply n x n: {tb * 1e3:.1f} ms "
      f"({2.0 * n ** 3 / tb / 1e12:.1f} TFLOP/s)")
