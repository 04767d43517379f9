"""Simultaneous shifted-system solvers dhsrq3 / chsrq3 (backsolve.py:350-388).

Same engine as the inverse-iteration seam with the solve-mode epilogue:
(H - lambda_l I) x_l = alpha_l b_l, robust (guarded, Omega = DBL_MAX/2/b_r)
or, with ``robust=False``, the unguarded tiled solve.
"""

from __future__ import annotations

import numpy as np

from .core import ConfigError, SolutionBlock, as_hessenberg
from .solver import MAX_TILE, raise_first_failure, solve_group, to_solution_block


def _driver(h, shifts, b, kind, *, b_r=None, b_c=32, workers=1, robust=True, mode="solve",
            stats=None, budget=None, workspace=None, device=None, compact_rotations=False):
    h = as_hessenberg(h)
    if not h.is_unreduced():
        raise ConfigError("matrix must be unreduced (nonzero subdiagonal)")
    n = h.n
    if b_r is None:
        b_r = min(MAX_TILE, n)
    if kind == "complex":
        lam = np.asarray(shifts, dtype=np.complex128).ravel()
        m = lam.size
        bb = np.asarray(b, dtype=np.complex128).reshape(n, m)
        B = np.empty((2 * m, n))
        B[0::2] = bb.real.T
        B[1::2] = bb.imag.T
        out, _ = solve_group(h, lam, None, B, b_r, robust=robust, mode=mode, b_c=b_c,
                             device=device, compact=compact_rotations)
    else:
        lam = np.asarray(shifts, dtype=np.float64).ravel()
        m = lam.size
        B = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n, m).T)
        out, _ = solve_group(h, None, lam, B, b_r, robust=robust, mode=mode, b_c=b_c,
                             device=device, compact=compact_rotations)
    if out.nfail:
        raise_first_failure(out.fail.cpu().numpy(), b_c, [(0, m)])
    return to_solution_block(out, n, robust=robust, want_cplx=(kind == "complex"))


def dhsrq3(h, shifts, b, **kw) -> SolutionBlock:
    """Solve (H - lam_l I) x_l = alpha_l b_l for real shifts (backsolve.py:376-383)."""
    return _driver(h, shifts, b, "real", **kw)


def chsrq3(h, shifts, b, **kw) -> SolutionBlock:
    """Complex-shift counterpart; b and x complex (n, m) (backsolve.py:386-388)."""
    return _driver(h, shifts, b, "complex", **kw)
