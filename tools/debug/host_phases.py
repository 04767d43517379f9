"""Per-phase device times of the host-buffer entry (pipelined, two in flight)
vs the device entry at config 5 -- where the e2e overhead goes."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.solver import HostGroupSolver  # noqa: E402

h, er, ec, b_r = bench.workload(5)
n = h.shape[0]
dev = torch.device("cuda", 0)
L = _lib.load()
pin = lambda shape: torch.empty(shape, dtype=torch.float64).pin_memory().numpy()
H = pin((n, n)).T
H[:] = h
lam = np.concatenate([ec.astype(np.complex128), er.astype(np.complex128)])
lre, lim, b = pin(lam.size), pin(lam.size), pin(n)
lre[:], lim[:] = lam.real, lam.imag
b[:] = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
hs = [HostGroupSolver(n, b_r, ec.size, er.size, dev) for _ in range(2)]
outs = [s.new_output(pinned=True) for s in hs]
stream = torch.cuda.current_stream(dev)


def run(k, timing):
    L.hsrq_set_timing(1 if timing else 0)
    prev = None
    for s in range(k):
        t = hs[s % 2].launch(H, lre, lim, b, True, outs[s % 2], stream=stream, wait=False)
        if prev is not None:
            hs[(s - 1) % 2].wait_ticket(prev, outs[(s - 1) % 2])
        prev = t
    hs[(k - 1) % 2].wait_ticket(prev, outs[(k - 1) % 2])
    L.hsrq_set_timing(0)


run(2, False)
pt = np.zeros(5)
L.hsrq_phase_times(ctypes.c_void_p(pt.ctypes.data))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
run(4, True)
e1.record(stream)
torch.cuda.synchronize()
L.hsrq_phase_times(ctypes.c_void_p(pt.ctypes.data))
print("host pipelined ms/step", e0.elapsed_time(e1) / 4, "phases (diag, panel, bt, setup, scalars)",
      np.round(pt / 4, 2).tolist())

# compute-stream span of each solve: events recorded right after each enqueue
evs = []
prev = None
for s_ in range(4):
    t = hs[s_ % 2].launch(H, lre, lim, b, True, outs[s_ % 2], stream=stream, wait=False)
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    evs.append(e)
    if prev is not None:
        hs[(s_ - 1) % 2].wait_ticket(prev, outs[(s_ - 1) % 2])
    prev = t
hs[3 % 2].wait_ticket(prev, outs[3 % 2])
torch.cuda.synchronize()
print("compute-stream span per solve (ms):", [round(evs[i - 1].elapsed_time(evs[i]), 1) for i in range(1, 4)])
