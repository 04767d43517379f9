"""Does hsrq_solve_group_host overlap the H upload with the sweep? (config 5)"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import instances  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver, HostGroupSolver  # noqa: E402

h = instances.make_h(5)
sel = instances.shifts(5)
er, ec = np.sort(sel[sel.imag == 0].real), sel[sel.imag > 0]
n = h.shape[0]
dev = torch.device("cuda", 0)
rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
pin = lambda shape: torch.empty(shape, dtype=torch.float64).pin_memory().numpy()
hh = pin((n, n)).T
hh[:] = h
lam = np.concatenate([ec, er.astype(complex)])
lre, lim, b = pin(lam.size), pin(lam.size), pin(n)
lre[:], lim[:], b[:] = lam.real, lam.imag, rho
hs = HostGroupSolver(n, 128, ec.size, er.size, dev)
out = hs.new_output(pinned=True)
st = torch.cuda.current_stream()
hs.launch(hh, lre, lim, b, True, out)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hs.launch(hh, lre, lim, b, True, out)
    t1 = time.perf_counter()
    print("host entry wall ms", round((t1 - t0) * 1e3, 1), flush=True)
# plain H2D and D2H of 2 GB
hd = torch.empty((n, n), dtype=torch.float64, device=dev)
src = torch.from_numpy(hh.T)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hd.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("H2D 2GB ms", round((t1 - t0) * 1e3, 1))
xd = torch.empty((2 * ec.size + er.size, n), dtype=torch.float64, device=dev)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    torch.from_numpy(out.X).copy_(xd, non_blocking=True)
    torch.cuda.synchronize()
    print("D2H X ms", round((time.perf_counter() - t0) * 1e3, 1))
gs = GroupSolver(DeviceHessenberg(HessenbergMatrix(h), dev), 128, ec.size, er.size)
gs.set_shifts(ec, er)
start = torch.full((n,), rho, dtype=torch.float64, device=dev)
gs.launch(start, True)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gs.launch(start, True)
    torch.cuda.synchronize()
    print("device entry wall ms", round((time.perf_counter() - t0) * 1e3, 1))
