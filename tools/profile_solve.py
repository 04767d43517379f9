"""One inverse-iteration solve attempt of a BASELINE config on cuda:0 (for ncu).

With HSRQ_LIB_VARIANT=counters it loads the diagnostics build
(libhsrq_b200_counters.so, ``_build.build(variant="counters",
defines=["HSRQ_COUNTERS"])``) and prints how often each guard path ran.
"""
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
ap.add_argument("--diag", default=None,
                help="force the diagonal variant: dp,dwr,dwc,wsr,wsc (hsrq_tune_diag)")
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
import ctypes
from paper_2101_05063_b200 import _lib
L = _lib.load()
if a.diag:
    L.hsrq_tune_diag(*[int(v) for v in a.diag.split(",")])
nf = gs.launch(start, True)  # warm-up
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(max(1, a.reps)):
    gs.launch(start, True, sync=False)
e1.record()
torch.cuda.synchronize()
print("solve ms (pipelined, no per-phase timing):", round(e0.elapsed_time(e1) / max(1, a.reps), 2))
L.hsrq_set_timing(1)
for _ in range(a.reps):
    nf = gs.launch(start, True)
torch.cuda.synchronize()
pt = np.zeros(5)
L.hsrq_phase_times(ctypes.c_void_p(pt.ctypes.data))
pt /= max(1, a.reps)
L.hsrq_set_timing(0)
print("failed", nf, "phase ms (diag, panel, backtransform, setup, scalars):", np.round(pt, 2).tolist())
cnt = np.zeros(32, dtype=np.int64)
_lib.load().hsrq_debug_counters(ctypes.c_void_p(cnt.ctypes.data), 1)
names = ["r_g1_fire", "r_g2_fire", "c_g1_exact", "c_g1_fire", "c_g2_exact", "c_g2_fire", "r_steps",
         "c_steps", "scal_items", "scal_exact1", "scal_exact2", "panel_s3_exact_cta",
         "c_g2_exact_warpsteps", "c_g2_full_warpsteps", "c_g2_mismatch", "c_g2_invalid",
         "wi_xmod", "wi_rmod", "wi_xr_mod", "wi_xr_ax_mod", "wi_ax_exact", "c_g2_e0",
         "wi_xbm_gt_omega", "wi_rx_gt_omega", "wi_ax_gt1"]
print({nm: int(v) for nm, v in zip(names, cnt)})
