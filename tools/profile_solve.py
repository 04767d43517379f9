"""One inverse-iteration solve attempt of a BASELINE config on cuda:0 (for ncu)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import instances  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
h = instances.make_h(a.config)
sel = instances.shifts(a.config)
er, ec = np.sort(sel[sel.imag == 0].real), sel[sel.imag > 0]
b_r = {1: 32, 2: 64}.get(a.config, 128)
hm = HessenbergMatrix(h)
dev = torch.device("cuda", 0)
gs = GroupSolver(DeviceHessenberg(hm, dev), b_r, ec.size, er.size)
gs.set_shifts(ec, er)
start = torch.full((hm.n,), np.finfo(float).eps * hm.infinity_norm(), dtype=torch.float64, device=dev)
for _ in range(a.reps):
    nf = gs.launch(start, True)
torch.cuda.synchronize()
print("failed", nf)
import ctypes
from paper_2101_05063_b200 import _lib
cnt = np.zeros(16, dtype=np.int64)
_lib.load().hsrq_debug_counters(ctypes.c_void_p(cnt.ctypes.data), 1)
names = ["r_g1_fire", "r_g2_fire", "c_g1_exact", "c_g1_fire", "c_g2_exact", "c_g2_fire", "r_steps",
         "c_steps", "scal_items", "scal_exact1", "scal_exact2", "panel_s3_exact_cta"]
print({nm: int(v) for nm, v in zip(names, cnt)})
