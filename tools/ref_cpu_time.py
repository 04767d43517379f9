"""Time the reference's own CPU path (hessrq's numba _solve_group, from
baseline/_ref) at config 5 on this host: one attempt over a sample of shifts,
workers=1 and workers=cores, beside the C oracle port."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import hessrq
    from hessrq.core import TileGrid, as_hessenberg
    from hessrq.inviter import InviterConfig, _solve_group

    import instances

    assert hessrq.backend_name() == "numba"
    nr, nc = int(sys.argv[1]), int(sys.argv[2])
    h = instances.make_h(5)
    sel = instances.shifts(5)
    er = sel[sel.imag == 0].real
    ec = sel[sel.imag > 0]
    rng = np.random.default_rng(1)
    sr = er[rng.choice(er.size, nr, replace=False)]
    sc = ec[rng.choice(ec.size, nc, replace=False)]
    hm = as_hessenberg(h)
    n = hm.n
    grid = TileGrid(n, 128)
    rho = np.finfo(float).eps * hm.infinity_norm()
    # JIT warm-up on a small problem
    hs = as_hessenberg(instances.random_hessenberg(300, 1))
    g2 = TileGrid(300, 128)
    for cp, lam in ((False, np.array([0.5, 0.7])), (True, np.array([0.5 + 1j, 0.2 + 0.3j]))):
        _solve_group(hs, g2, lam, np.ones((300, 2), dtype=complex if cp else float),
                     InviterConfig(b_r=128), None, cp)
    cores = os.cpu_count()
    for workers in (1, cores):
        cfg = InviterConfig(b_r=128, workers=workers)
        t0 = time.perf_counter()
        rr = _solve_group(hm, grid, sr, np.repeat(rho * np.ones((n, 1)), nr, 1), cfg, None, False)
        t1 = time.perf_counter()
        rc = _solve_group(hm, grid, sc, np.repeat(rho * np.ones((n, 1)), nc, 1).astype(complex), cfg,
                          None, True)
        t2 = time.perf_counter()
        conv = int(np.sum(rr.norms > 0.1 / np.sqrt(n)) + np.sum(rc.norms > 0.1 / np.sqrt(n)))
        print(f"workers={workers}: {nr} real {t1 - t0:.2f} s ({(t1 - t0) / nr:.3f} s/shift), "
              f"{nc} complex {t2 - t1:.2f} s ({(t2 - t1) / nc:.3f} s/shift); converged {conv}/{nr + nc}",
              flush=True)


if __name__ == "__main__":
    main()
