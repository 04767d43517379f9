"""Henry's single-sweep RQ solve on the GPU: the reference's baseline solver.

Mirrors ``henry_rq_solve`` (hessrq reference.py:21-60): same arguments
(H, a scalar shift or a batch, a right-hand side per shift), same result
shapes and the same exceptions with the same ``shift_index`` /
``local_index``; the arithmetic runs in ``k_henry_real`` / ``k_henry_cplx``
(csrc/hsrq_henry.cuh) through ``hsrq_henry_solve`` (include/hsrq.h) and is
bit-identical to the reference kernels (numba_backend.py:830-923).

One deliberate difference: the reference's complex path fails on success
under its numba backend (``henry_solve_complex`` falls off its end and
returns None, which ``unpack_status`` rejects with TypeError); here it
returns the solution, as the reference's docstring and numpy backend do.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import HessrqError, SingularSystemError, StructuralViolationError, as_hessenberg
from .solver import DeviceHessenberg, default_device

_KIND_DEGENERATE = 1


def _unpack(status):
    status = int(status)
    return status >> 42, (status >> 21) & ((1 << 21) - 1), status & ((1 << 21) - 1)


def henry_solve_device(dh, lam, X, cplx, stream=None):
    """Enqueue-and-wait on device tensors: ``lam`` (m,) float64 or (m, 2)
    float64 (re, im); ``X`` (m, n) float64 or (m, n, 2) float64, row l =
    column l of the right-hand side, overwritten by the solution.  Returns
    the packed status (0 = ok)."""
    lib = _lib.load()
    n, m = dh.n, int(lam.shape[0])
    ws_bytes = int(lib.hsrq_henry_workspace_bytes(n, m, int(cplx)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dh.device)
    stream = stream or torch.cuda.current_stream(dh.device)
    st = lib.hsrq_henry_solve(
        ctypes.c_void_p(dh.t.data_ptr()), dh.ldh, n, ctypes.c_void_p(lam.data_ptr()), m,
        int(cplx), ctypes.c_void_p(X.data_ptr()), n, None, ctypes.c_void_p(ws.data_ptr()),
        ws_bytes, ctypes.c_void_p(stream.cuda_stream))
    if st < 0:
        raise RuntimeError(f"hsrq_henry_solve failed ({st}): {_lib.last_error()}")
    return int(st)


def henry_rq_solve(h, lam, b, device=None):
    """Solve (H - lam I) x = b in one merged factor-and-substitute sweep.

    ``lam`` may be a scalar or a batch; complex shifts run in full complex
    arithmetic.  H is never modified (reference.py:21-60).
    """
    h = as_hessenberg(h)
    n = h.n
    lam_arr = np.atleast_1d(np.asarray(lam))
    single_shift = np.isscalar(lam) or np.asarray(lam).ndim == 0
    cplx = np.iscomplexobj(lam_arr)
    m = lam_arr.shape[0]
    bb = np.asarray(b)
    single_col = bb.ndim == 1
    dev = device or default_device()
    dh = DeviceHessenberg.of(h, dev)
    if cplx:
        xb = np.asarray(bb, dtype=np.complex128).reshape(n, m)
        Xh = np.ascontiguousarray(xb.T)  # row l = column l
        X = torch.from_numpy(Xh.view(np.float64).reshape(m, n, 2)).to(dev)
        lam_t = torch.from_numpy(np.ascontiguousarray(lam_arr, dtype=np.complex128)
                                 .view(np.float64).reshape(m, 2)).to(dev)
    else:
        xb = np.asarray(bb, dtype=np.float64).reshape(n, m)
        X = torch.from_numpy(np.ascontiguousarray(xb.T)).to(dev)
        lam_t = torch.from_numpy(np.ascontiguousarray(lam_arr, dtype=np.float64)).to(dev)
    status = henry_solve_device(dh, lam_t, X, cplx)
    if status != 0:
        kind, l, row = _unpack(status)
        if kind == _KIND_DEGENERATE:
            raise StructuralViolationError(
                f"zero pivot pair at row {row} (matrix not unreduced?)")
        raise SingularSystemError(
            f"zero pivot phi for shift {l} at row {row}", shift_index=l, local_index=row)
    Xc = X.cpu().numpy()
    if cplx:
        x = np.ascontiguousarray(Xc.reshape(m, n, 2).view(np.complex128).reshape(m, n).T)
    else:
        x = np.ascontiguousarray(Xc.T)
    if single_col and single_shift:
        return x[:, 0]
    return x


__all__ = ["henry_rq_solve", "henry_solve_device", "HessrqError"]
