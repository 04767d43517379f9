"""Eager vs CUDA-graph replay of one solve group (hsrq_graph_capture) on a
small, launch-bound problem.  python tools/graph_time.py n m b_r"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import instances  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

n, m, b_r = (int(v) for v in sys.argv[1:4])
h = instances.random_hessenberg(n, 0)
ev = np.linalg.eigvals(h)
er, ec = ev[ev.imag == 0].real[: m // 2], ev[ev.imag > 0][: m // 2]
dev = torch.device("cuda", 0)
dh = DeviceHessenberg(HessenbergMatrix(h), dev)
b = torch.full((n,), 1e-3, dtype=torch.float64, device=dev)
gs = GroupSolver(dh, b_r, ec.size, er.size)
gs.set_shifts(ec, er)
for _ in range(3):
    gs.launch(b, True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
e0.record()
for _ in range(reps):
    gs.launch(b, True, sync=False)
e1.record()
torch.cuda.synchronize()
eager = e0.elapsed_time(e1) / reps
gs.capture(b, True)
for _ in range(3):
    gs.replay(sync=False)
e0.record()
for _ in range(reps):
    gs.replay(sync=False)
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / reps
print(f"n={n} shifts={ec.size}c+{er.size}r b_r={b_r}: eager {eager:.3f} ms, graph replay {graph:.3f} ms "
      f"({eager / graph:.2f}x)")
