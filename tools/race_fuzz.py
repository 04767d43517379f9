"""Race check by schedule fuzzing (compute-sanitizer is closed on the GPU pool).

Runs a fixed set of solves -- every diagonal-sweep variant (one-warp and
warp-pair, real and complex, DP 4 ... 32), the lookahead schedule (sweep
beside the panel on other streams), every backtransform width, and the Henry
sweep -- with start vectors at 1e300 so every guard path fires, and writes
all outputs to an .npz.  Run once with the production library and then,
several times, with the schedule-fuzzing build (``-DHSRQ_FUZZ``:
pseudo-random threads sleep up to ~2 us after every barrier, see
csrc/hsrq_device.cuh); any shared-memory value consumed without the barrier
that orders it changes a result bit:

  python tools/race_fuzz.py --save /tmp/prod.npz
  HSRQ_LIB_VARIANT=fuzz python tools/race_fuzz.py --compare /tmp/prod.npz --reps 3
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
from paper_2101_05063_b200 import _lib  # noqa: E402
from paper_2101_05063_b200.core import HessenbergMatrix  # noqa: E402
from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver  # noqa: E402

VARIANTS = [(4, 4, 2, 0, 2), (4, 4, 2, 0, 0), (4, 4, 2, 2, 2), (8, 6, 4, 0, 0), (8, 6, 4, 2, 2),
            (16, 16, 16, 0, 0), (16, 16, 16, 2, 2), (32, 16, 16, 0, 0), (32, 16, 16, 4, 4),
            (16, 16, 16, 0, 0, 8), (32, 16, 16, 0, 0, 4)]  # 6th: rotation-ahead pairs
CASES = [(300, 64, 3, 8, 16), (515, 100, 6, 8, 40)]  # n, b_r, seed, real, complex


def run_all():
    dev = torch.device("cuda", 0)
    L = _lib.load()
    res = {}
    for ci, (n, b_r, seed, nr, nc) in enumerate(CASES):
        h = instances.random_hessenberg(n, seed)
        ev = np.linalg.eigvals(h)
        er = ev[ev.imag == 0].real[:nr]
        ec = ev[ev.imag > 0][:nc]
        dh = DeviceHessenberg(HessenbergMatrix(h), dev)
        B = torch.full((n,), 1e300, dtype=torch.float64, device=dev)
        for vi, v in enumerate(VARIANTS):
            for la in ("0", "1"):
                L.hsrq_tune_diag(*v[:5])
                L.hsrq_tune_diag_rx(v[5] if len(v) > 5 else 0)
                os.environ["HSRQ_BT_G"] = str((4, 8, 16, 32)[vi % 4])
                os.environ["HSRQ_LOOKAHEAD"] = la
                gs = GroupSolver(dh, b_r, ec.size, er.size)
                gs.set_shifts(ec, er)
                nf = gs.launch(B, True)
                key = f"c{ci}_v{vi}_la{la}"
                for name in ("X", "seg_exp", "alpha_exp", "norms", "c_re", "c_im", "s", "fail"):
                    res[f"{key}_{name}"] = getattr(gs, name).cpu().numpy().copy()
                res[f"{key}_nfail"] = np.array(nf)
        # Henry's single sweep (one CTA per shift, one barrier per step)
        from paper_2101_05063_b200 import henry

        lam = np.concatenate([er, ec])
        xh = henry.henry_rq_solve(h, lam, np.ones((n, lam.size), dtype=complex))
        res[f"c{ci}_henry"] = np.asarray(xh)
    for k in ("HSRQ_BT_G", "HSRQ_LOOKAHEAD"):
        os.environ.pop(k, None)
    L.hsrq_tune_diag(0, 0, 0, -1, -1)
    L.hsrq_tune_diag_rx(-1)
    torch.cuda.synchronize()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--save")
    ap.add_argument("--compare")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    variant = os.environ.get("HSRQ_LIB_VARIANT", "production")
    if a.save:
        np.savez(a.save, **run_all())
        print(f"saved {a.save} ({variant})")
        return 0
    want = np.load(a.compare)
    bad = 0
    for r in range(a.reps):
        got = run_all()
        diff = [k for k in want.files
                if not np.array_equal(np.atleast_1d(want[k]).view(np.uint8),
                                      np.atleast_1d(got[k]).view(np.uint8))]
        bad += len(diff)
        print(f"rep {r} ({variant}): {len(want.files)} arrays, {len(diff)} differ"
              + (f": {diff[:8]}" if diff else ""), flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
