"""Does the order of the complex shifts (which 8 share a warp in the DP = 4
sweep) change the diag time?  The warp takes the guard-2 exact pass when any
of its shifts needs it."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import bench  # noqa: E402
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

h, er, ec, b_r = bench.workload(5)
hm = HessenbergMatrix(h)
dev = torch.device("cuda", 0)
dh = DeviceHessenberg(hm, dev)
L = _lib.load()
start = torch.full((hm.n,), np.finfo(float).eps * hm.infinity_norm(), dtype=torch.float64, device=dev)
gs = GroupSolver(dh, b_r, ec.size, er.size)
orders = {"lapack": np.arange(ec.size), "abs": np.argsort(np.abs(ec)), "re": np.argsort(ec.real),
          "im": np.argsort(ec.imag), "arg": np.argsort(np.angle(ec))}
for name, perm in orders.items():
    gs.set_shifts(ec[perm], er)
    gs.launch(start, True)
    L.hsrq_phase_times(ctypes.c_void_p(np.zeros(5).ctypes.data))
    L.hsrq_set_timing(1)
    gs.launch(start, True)
    L.hsrq_set_timing(0)
    pt = np.zeros(5)
    L.hsrq_phase_times(ctypes.c_void_p(pt.ctypes.data))
    print(name, "diag", round(pt[0], 1), "total", round(pt.sum(), 1), flush=True)
