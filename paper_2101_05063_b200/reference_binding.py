"""Binding of the B200 seam into the reference package itself.

``solve_group_b200`` has the signature and contract of hessrq's
``_solve_group(h, grid, eigs, b, config, workspace, cplx)``
(inviter.py:91-106): it takes the reference's HessenbergMatrix / TileGrid /
InviterConfig objects and numpy arrays, runs one robust tiled solve in
eigvec mode on the GPU (libhsrq_b200 through solver.solve_group), and returns
the reference's own ``SolutionBlock`` (x, alpha, segment scales, norms) --
raising the reference's own ``SingularSystemError`` /
``StructuralViolationError`` for the first failure in the reference's order
(tiled_reduce before the substitution, batches of ``config.b_c``, tile
columns right to left, rows bottom-up: solver.raise_first_failure), with its
``shift_index`` / ``local_index``.  ``install(hessrq.inviter)`` swaps it in,
so the reference's ``_iterate`` / ``dhsrq3in`` / ``chsrq3in`` / ``hsrq3in``
(restarts, convergence, ordering: unchanged reference code) run on the B200
kernels -- the one-line switch INTEGRATION.md describes.
"""

from __future__ import annotations

import sys

import numpy as np

from . import core as _core
from .solver import DeviceHessenberg, raise_first_failure, solve_group

_DMAX = float(np.finfo(np.float64).max)


def _ref_module(obj, name):
    """The reference's class ``name`` from the module ``obj``'s type lives in
    (hessrq.core), or this package's stand-in."""
    mod = sys.modules.get(type(obj).__module__)
    return getattr(mod, name, None) or getattr(_core, name)


def _device_h(h):
    """Cached device copy of a reference HessenbergMatrix (its data is
    read-only, core.py:74, so the cache cannot go stale)."""
    d = getattr(h, "_b200_device", None)
    if d is None:
        d = DeviceHessenberg.upload(np.asarray(h.data))
        try:
            h._b200_device = d
        except AttributeError:  # pragma: no cover - slotted stand-ins
            pass
    return d


def solve_group_b200(h, grid, eigs, b, config, workspace, cplx):
    """hessrq ``_solve_group`` (inviter.py:91-106) on the GPU."""
    n = h.n
    lam = np.asarray(eigs)
    m = lam.shape[0]
    bb = np.asarray(b).reshape(n, m)
    # _iterate passes one start vector repeated per column (inviter.py:127-133)
    if m and np.all(bb == bb[:, :1]):
        B = np.ascontiguousarray(bb[:, 0].real, dtype=np.float64)
    elif cplx:
        B = np.empty((2 * m, n))
        B[0::2] = bb.real.T
        B[1::2] = bb.imag.T
    else:
        B = np.ascontiguousarray(bb.real.T, dtype=np.float64)
    if workspace is not None and hasattr(workspace, "peak_crossover_reals"):
        workspace.peak_crossover_reals = max(workspace.peak_crossover_reals,
                                             n * grid.N * m * (2 if cplx else 1))
    dh = _device_h(h)
    if cplx:
        out, _ = solve_group(dh, lam.astype(np.complex128), None, B, grid.b_r, robust=True,
                             mode="eigvec", b_c=config.b_c)
    else:
        out, _ = solve_group(dh, None, lam.astype(np.float64), B, grid.b_r, robust=True,
                             mode="eigvec", b_c=config.b_c)
    if out.nfail:
        # the reference's executor re-raises the kernel's error as TaskError with
        # the failing node (scheduler.py:182-187, 211-214): the same here, in the
        # reference's own classes
        try:
            raise_first_failure(out.fail.cpu().numpy(), config.b_c, [(0, m)], n_tiles=grid.N)
        except _core.TaskError as e:
            if isinstance(e, _core.SingularSystemError):
                cause = _ref_module(h, "SingularSystemError")(
                    str(e.cause), shift_index=e.shift_index, local_index=e.local_index)
            else:
                cause = _ref_module(h, "StructuralViolationError")(str(e.cause))
            sched = sys.modules.get(type(h).__module__.rsplit(".", 1)[0] + ".scheduler")
            if sched is None or not hasattr(sched, "TaskError"):
                raise cause from None
            node = sched.TaskNode(e.node.kind, e.node.coords, seq=e.node.seq)
            raise sched.TaskError(node, cause) from cause
    X = out.X.cpu().numpy()
    x = (X[0::2] + 1j * X[1::2]).T.copy() if cplx else X.T.copy()
    aexp = out.alpha_exp.cpu().numpy()
    seg = out.seg_exp.cpu().numpy()
    SolutionBlock = _ref_module(h, "SolutionBlock")
    ScalingMatrix = _ref_module(h, "ScalingMatrix")
    # the reference's doubles: ldexp(1, e) (0 where its scale would underflow)
    return SolutionBlock(x=x, alpha=np.ldexp(1.0, aexp),
                         segment_scales=ScalingMatrix(np.ldexp(1.0, seg)),
                         norms=out.norms.cpu().numpy())


def install(inviter_module):
    """Route ``inviter_module._solve_group`` (hessrq.inviter) to the GPU;
    returns the original for ``uninstall``."""
    orig = inviter_module._solve_group
    inviter_module._solve_group = solve_group_b200
    return orig


def uninstall(inviter_module, orig):
    inviter_module._solve_group = orig
