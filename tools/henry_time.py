"""Time the GPU Henry single sweep (hsrq_henry_solve) on config-like inputs.
python tools/henry_time.py n m_real m_cplx"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2101_05063_b200.henry import henry_solve_device  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg  # noqa: E402

n, mr, mc = (int(v) for v in sys.argv[1:4])
rng = np.random.default_rng(0)
h = np.triu(rng.standard_normal((n, n)))
h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
dh = DeviceHessenberg(h)
for cplx, m in ((False, mr), (True, mc)):
    if m == 0:
        continue
    lam = rng.uniform(-3, 3, m) + (1j * rng.uniform(0.1, 2, m) if cplx else 0)
    if cplx:
        lam_t = torch.from_numpy(lam.astype(np.complex128).view(np.float64).reshape(m, 2)).cuda()
        X0 = torch.ones((m, n, 2), dtype=torch.float64, device="cuda")
    else:
        lam_t = torch.from_numpy(lam).cuda()
        X0 = torch.ones((m, n), dtype=torch.float64, device="cuda")
    for rep in range(3):
        X = X0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = henry_solve_device(dh, lam_t, X, cplx)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    # traffic model: per row-step v,x RMW + h read (L2), bytes
    w = 2 if cplx else 1
    rowsteps = n * (n - 1) / 2.0
    print(f"n={n} {'complex' if cplx else 'real'} m={m}: {ms:.1f} ms  status={st}  "
          f"{ms / m:.3f} ms/shift  row-step traffic {rowsteps * m * 8 * (4 * w + 1) / ms / 1e6:.0f} GB/s")
