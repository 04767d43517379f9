"""Small solves that drive every diagonal-sweep variant (one-warp and
warp-pair, real and complex, DP 4 ... 32), the panel, k_scalars and every
backtransform width, for compute-sanitizer runs (one tool per call):

  compute-sanitizer --tool racecheck --kernel-name kns=k_diag python tools/sanitize_case.py
  compute-sanitizer --tool memcheck python tools/sanitize_case.py

The warp-pair sweeps exchange per-step values through shared memory slots
double-buffered by step parity and join with named barriers (bar.sync id, 64;
csrc/hsrq_diag_ws.cuh); racecheck reports any hazard on those slots.
Start vectors at 1e300 make every guard (and its rescaling / exact
certification path) fire."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import instances  # noqa: E402
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

VARIANTS = [(4, 4, 2, 2, 2), (4, 4, 2, 0, 0), (8, 6, 4, 2, 2), (16, 16, 16, 2, 2),
            (32, 16, 16, 4, 4), (32, 16, 16, 0, 0)]


def main():
    quick = "--quick" in sys.argv
    dev = torch.device("cuda", 0)
    L = _lib.load()
    n, b_r = (260, 64) if quick else (300, 64)
    h = instances.random_hessenberg(n, 3)
    ev = np.linalg.eigvals(h)
    er = ev[ev.imag == 0].real[:8]
    ec = ev[ev.imag > 0][:16]
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    B = torch.full((n,), 1e300, dtype=torch.float64, device=dev)
    base = None
    for i, v in enumerate(VARIANTS):
        L.hsrq_tune_diag(*v)
        os.environ["HSRQ_BT_G"] = str((4, 8, 16, 32)[i % 4])
        gs = GroupSolver(dh, b_r, ec.size, er.size)
        gs.set_shifts(ec, er)
        nf = gs.launch(B, True)
        x = gs.X.cpu().numpy()
        if base is None:
            base = x
        ok = np.array_equal(base.view(np.int64), x.view(np.int64))
        print(f"variant {v} G={os.environ['HSRQ_BT_G']}: nfail={nf} bitwise_same={ok}", flush=True)
        assert nf == 0 and ok
    torch.cuda.synchronize()
    print("sanitize case done")


if __name__ == "__main__":
    main()
