"""Per-rank time of the config-5 sweep for a world size W, measured on ONE GPU
by running rank 0's shard alone (ranks are independent: no collective inside
the sweep, parallel.py) -- a proxy for the strong-scaling behaviour.
python tools/shard_time.py W [W ...]   (HSRQ_DIAG=DP,DWR,DWC selects a variant;
SHARD_ONLY=real|cplx keeps one kind of shift)"""
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

h, er, ec, b_r = bench.workload(5)
hm = HessenbergMatrix(h)
dev = torch.device("cuda", 0)
dh = DeviceHessenberg(hm, dev)
L = _lib.load()
start = torch.full((hm.n,), np.finfo(float).eps * hm.infinity_norm(), dtype=torch.float64, device=dev)
for W in (int(w) for w in sys.argv[1:]):
    my_r, my_c = bench.partition(er, ec, 0, W)
    only = os.environ.get("SHARD_ONLY")  # "real" / "cplx": drop the other kind (diagnostics)
    if only == "real":
        my_c = my_c[:0]
    elif only == "cplx":
        my_r = my_r[:0]
    gs = GroupSolver(dh, b_r, my_c.size, my_r.size)
    gs.set_shifts(my_c, my_r)
    gs.launch(start, True)
    graph = os.environ.get("HSRQ_GRAPH") == "1"  # replay the sweep as one CUDA graph
    if graph:
        gs.capture(start, True)
        gs.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        if graph:
            gs.replay(sync=False)
        else:
            gs.launch(start, True, sync=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    L.hsrq_set_timing(1)
    nf = gs.launch(start, True)
    L.hsrq_set_timing(0)
    pt = np.zeros(5)
    L.hsrq_phase_times(ctypes.c_void_p(pt.ctypes.data))
    print(f"W={W} diag={os.environ.get('HSRQ_DIAG', 'default')} shard {my_r.size}r+{my_c.size}c: "
          f"{ms:.1f} ms/solve; phases diag {pt[0]:.1f} panel {pt[1]:.1f} scalars {pt[4]:.1f} "
          f"bt {pt[2]:.1f} failed {nf}", flush=True)
    del gs
    torch.cuda.empty_cache()
