"""Per-step phase breakdown of the rotation-ahead complex sweep
(k_diag_cplx_rx) at a config-5 shard (HSRQ_LIB_VARIANT=stepprof):
python tools/rx_profile.py W DP NP"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
import bench  # noqa: E402
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

W, DP, NP = (int(v) for v in sys.argv[1:4])
R = ["row kp reads + prefetch", "two hypots", "divisions, pivot, rb", "R column + v update",
     "maxima, slot, prefetch wait", "pair barrier wait"]
X = ["slot reads", "guard 1 + x_kp read", "complex division", "guard 2 (bound, cert, rescale)",
     "x update + maxima", "pair barrier wait"]
h, er, ec, b_r = bench.workload(5)
dev = torch.device("cuda", 0)
dh = DeviceHessenberg(HessenbergMatrix(h), dev)
L = _lib.load()
L.hsrq_tune_diag(DP, 16, 16, 0, 0)
L.hsrq_tune_diag_rx(NP)
my_r, my_c = bench.partition(er, ec, 0, W)
gs = GroupSolver(dh, b_r, my_c.size, 0)
gs.set_shifts(my_c, [])
start = torch.full((dh.n,), np.finfo(float).eps * dh.norm_inf, dtype=torch.float64, device=dev)
gs.launch(start, True)
out = np.zeros(16, dtype=np.int64)
L.hsrq_debug_stepprof(ctypes.c_void_p(out.ctypes.data), 1)
gs.launch(start, True)
L.hsrq_debug_stepprof(ctypes.c_void_p(out.ctypes.data), 1)
steps = max(1, out[15] * 127)
print(f"W={W} DP={DP} NP={NP}: {my_c.size} complex shifts; cycles per step (warp pair 0 of each CTA)")
# X-warp marks: [6..11] map 5 -> slot reads, 0 guard1, 1 cdiv, 2 guard2, 3 update, 4 barrier
xmap = {5: 0, 0: 1, 1: 2, 2: 3, 3: 4, 4: 5}
for j in range(6):
    print(f"  R {R[j]:32s} {out[j] / steps:7.0f}    X {X[xmap[j] if False else j]:34s}", end="")
    print(f" {out[6 + [5, 0, 1, 2, 3, 4][j]] / steps:7.0f}")
print(f"  R total {out[:6].sum() / steps:7.0f}   X total {out[6:12].sum() / steps:7.0f}")
