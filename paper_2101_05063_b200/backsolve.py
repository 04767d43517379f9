"""Simultaneous shifted-system solvers dhsrq3 / chsrq3 (backsolve.py:350-388).

Same engine as the inverse-iteration seam with the solve-mode epilogue:
(H - lambda_l I) x_l = alpha_l b_l, robust (guarded, Omega = DBL_MAX/2/b_r)
or, with ``robust=False``, the unguarded tiled solve.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .core import ConfigError, SolutionBlock, as_hessenberg
from .solver import MAX_TILE, raise_first_failure, solve_group, to_solution_block


_DMAX = float(np.finfo(np.float64).max)


def _driver(h, shifts, b, kind, *, b_r=None, b_c=32, workers=1, robust=True, mode="solve",
            stats=None, budget=None, workspace=None, device=None, compact_rotations=False):
    """``workers`` is accepted and ignored (every shift runs concurrently on the
    device); ``budget`` (an OverflowBudget-like object with ``.omega``,
    overflow.py:31-47) replaces the default DBL_MAX/2/b_r; ``workspace``
    (core.Workspace-like) gets the reference's cross-over high-water mark
    (reduce.py:63-75: n * N * cols reals)."""
    h = as_hessenberg(h)
    if not h.is_unreduced():
        raise ConfigError("matrix must be unreduced (nonzero subdiagonal)")
    n = h.n
    if b_r is None:
        b_r = min(MAX_TILE, n)
    omega = None
    if budget is not None:
        omega = float(budget.omega)
        if not (0.0 < omega <= _DMAX / 2.0):
            raise ValueError(f"omega={omega} outside (0, maxfloat/2]")
    lib = None
    if stats is not None:  # per-phase device times for the RunStats counters
        from . import _lib

        lib = _lib.load()
        lib.hsrq_phase_times((ctypes.c_double * 5)())  # drop stale timings
        lib.hsrq_set_timing(1)
    try:
        out, m, cplx = _run(h, shifts, b, kind, n, b_r, b_c, robust, mode, device,
                            compact_rotations, omega)
    finally:
        if lib is not None:
            lib.hsrq_set_timing(0)
    if stats is not None:
        from . import flops
        from .benchcsv import GPU_PHASES, task_seconds

        ph = (ctypes.c_double * 5)()
        lib.hsrq_phase_times(ph)
        ex, fo = flops.task_flops(n, b_r, m, cplx)
        sec = task_seconds(dict(zip(GPU_PHASES, [v / 1e3 for v in ph])), ex)
        for t in flops.TASK_TYPES:
            stats.add(t, sec[t], ex[t], fo[t])
    if workspace is not None and hasattr(workspace, "peak_crossover_reals"):
        N = (n + b_r - 1) // b_r
        workspace.peak_crossover_reals = max(workspace.peak_crossover_reals,
                                             n * N * m * (2 if cplx else 1))
    if out.nfail:
        raise_first_failure(out.fail.cpu().numpy(), b_c, [(0, m)], n_tiles=(n + b_r - 1) // b_r)
    return to_solution_block(out, n, robust=robust, want_cplx=cplx)


def _run(h, shifts, b, kind, n, b_r, b_c, robust, mode, device, compact_rotations, omega=None):
    if kind == "complex":
        lam = np.asarray(shifts, dtype=np.complex128).ravel()
        m = lam.size
        bb = np.asarray(b, dtype=np.complex128).reshape(n, m)
        B = np.empty((2 * m, n))
        B[0::2] = bb.real.T
        B[1::2] = bb.imag.T
        out, _ = solve_group(h, lam, None, B, b_r, robust=robust, mode=mode, b_c=b_c,
                             device=device, compact=compact_rotations, omega=omega)
    else:
        lam = np.asarray(shifts, dtype=np.float64).ravel()
        m = lam.size
        B = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n, m).T)
        out, _ = solve_group(h, None, lam, B, b_r, robust=robust, mode=mode, b_c=b_c,
                             device=device, compact=compact_rotations, omega=omega)
    return out, m, kind == "complex"


def dhsrq3(h, shifts, b, **kw) -> SolutionBlock:
    """Solve (H - lam_l I) x_l = alpha_l b_l for real shifts (backsolve.py:376-383)."""
    return _driver(h, shifts, b, "real", **kw)


def chsrq3(h, shifts, b, **kw) -> SolutionBlock:
    """Complex-shift counterpart; b and x complex (n, m) (backsolve.py:386-388)."""
    return _driver(h, shifts, b, "complex", **kw)
