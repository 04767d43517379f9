"""Per-step phase breakdown of the one-warp complex diagonal sweep
(k_diag_cplx) for a config-5 shard: build the -DHSRQ_STEPPROF variant
(libhsrq_b200_stepprof.so) and run with HSRQ_LIB_VARIANT=stepprof.
python tools/step_profile.py W   (rank 0's W-way shard; DP from diag_pick, the
warp-pair kernel forced off so k_diag_cplx runs)"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

PHASES = ["prefetch issue + row kp reads", "two glibc hypots", "3 divisions, pivot, rotation store",
          "group maxima + guard 1", "complex pivot division", "guard-2 bound test",
          "guard-2 certification / exact / rescale", "row update (rows < kp-1)", "shifted row",
          "prefetch wait + warp barrier"]
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
h, er, ec, b_r = bench.workload(5)
dev = torch.device("cuda", 0)
dh = DeviceHessenberg(HessenbergMatrix(h), dev)
L = _lib.load()
L.hsrq_tune_diag(0, 0, 0, -1, 0)  # automatic DP, no warp pairs for the complex sweep
my_r, my_c = bench.partition(er, ec, 0, W)
my_r = my_r[:0]  # complex sweep only (no concurrent real sweep)
gs = GroupSolver(dh, b_r, my_c.size, my_r.size)
gs.set_shifts(my_c, my_r)
start = torch.full((hm_n := dh.n,), np.finfo(float).eps * dh.norm_inf, dtype=torch.float64, device=dev)
gs.launch(start, True)
out = np.zeros(16, dtype=np.int64)
L.hsrq_debug_stepprof(ctypes.c_void_p(out.ctypes.data), 1)
gs.launch(start, True)
L.hsrq_debug_stepprof(ctypes.c_void_p(out.ctypes.data), 1)
warps = out[15]
steps = warps * 127  # steps per full tile column (k = 128), approximately
tot = out[:10].sum()
print(f"W={W}: {my_c.size} complex shifts, profiled warp-sweeps {warps}, "
      f"{tot / max(steps, 1):.0f} cycles per step")
for i, name in enumerate(PHASES):
    print(f"  {name:42s} {out[i] / max(steps, 1):8.0f} cycles  {100 * out[i] / max(tot, 1):5.1f} %")
