"""Front end of the path on the GPU.

* ``householder_hessenberg(a)`` -- the reference's dense-to-Hessenberg
  reduction (testprob.py:146-174): returns (H, Q) with Q^T A Q = H, same
  reflectors, sign convention and skip rule, computed by
  ``hsrq_hessenberg_reduce`` (csrc/hsrq_hessenberg.cu, blocked DGEHRD
  scheme: level-2 panel + fp64 GEMM updates).
* ``backmultiply(Q, X)`` -- eigenvectors of H to eigenvectors of A,
  z = Q0 x, one fp64 GEMM.
* ``hsrq3in_dense(a, eigenvalues, config)`` -- the whole pipeline for a
  dense real A: reduce, the inverse-iteration path (``hsrq3in``) on H,
  back-multiply; the eigenvalues are those of A (= those of H).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .core import ConfigError, HessenbergMatrix
from .solver import default_device


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def hessenberg_device(A, want_q=True):
    """Reduce the device matrix ``A`` in place.  ``A``: (n, n) float64 CUDA
    tensor holding the matrix COLUMN-major (i.e. row r of the tensor is
    column r of the matrix, ``A_mat = A.T``).  Returns Q in the same
    convention (or None)."""
    lib = _lib.load()
    n = A.shape[0]
    # odd n: work in buffers with an even leading dimension, so every column stays
    # 16-byte aligned for the streaming kernels (15999 vs 16000: 4.8 s -> as 16000)
    ld = n + (n & 1)
    Aw = A if ld == n else torch.zeros((n, ld), dtype=torch.float64, device=A.device)
    if Aw is not A:
        Aw[:, :n] = A
    Q = torch.empty((n, ld), dtype=torch.float64, device=A.device) if want_q else None
    wsb = int(lib.hsrq_hessenberg_workspace_bytes(n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=A.device)
    r = lib.hsrq_hessenberg_reduce(ctypes.c_void_p(Aw.data_ptr()), ld,
                                   ctypes.c_void_p(Q.data_ptr()) if want_q else None, ld, n,
                                   ctypes.c_void_p(ws.data_ptr()), wsb, _stream(A.device))
    if r != 0:
        raise RuntimeError(f"hsrq_hessenberg_reduce failed ({r}): "
                           f"{lib.hsrq_hessenberg_last_error().decode()}")
    if Aw is not A:
        A.copy_(Aw[:, :n])
        if want_q:
            Q = Q[:, :n].contiguous()
    return Q


def householder_hessenberg(a, device=None):
    """Reduce a dense square matrix to upper Hessenberg form (testprob.py:146-174).

    Returns (H, Q) with Q orthogonal and Q.T @ A @ Q = H.  Columns whose
    below-subdiagonal part is already zero are skipped, so an input that is
    already Hessenberg comes back unchanged with Q = I.
    """
    a = np.array(a, dtype=np.float64)
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise ConfigError(f"expected square matrix, got {a.shape}")
    dev = device or default_device()
    A = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)  # rows = columns
    Q = hessenberg_device(A)
    return A.cpu().numpy().T.copy(), Q.cpu().numpy().T.copy()


def backmultiply_device(Q, X):
    """Z = Q X on the device.  Q: (n, n) tensor in the column-major convention
    of ``hessenberg_device``; X: (ncol, n) tensor, row c = column c.  Returns Z
    in X's convention."""
    lib = _lib.load()
    n = Q.shape[0]
    ncol = X.shape[0]
    Z = torch.empty_like(X)
    r = lib.hsrq_backmultiply(ctypes.c_void_p(Q.data_ptr()), n, n, ctypes.c_void_p(X.data_ptr()),
                              n, ncol, ctypes.c_void_p(Z.data_ptr()), n, _stream(Q.device))
    if r != 0:
        raise RuntimeError(f"hsrq_backmultiply failed ({r})")
    return Z


def backmultiply(q, x, device=None):
    """z = Q x for host arrays: q (n, n), x (n, m) real or complex."""
    dev = device or default_device()
    q = np.asarray(q, dtype=np.float64)
    x = np.asarray(x)
    cplx = np.iscomplexobj(x)
    Qt = torch.from_numpy(np.ascontiguousarray(q.T)).to(dev)
    cols = [x.real, x.imag] if cplx else [x]
    outs = []
    for part in cols:
        X = torch.from_numpy(np.ascontiguousarray(np.asarray(part, dtype=np.float64).T)).to(dev)
        outs.append(backmultiply_device(Qt, X).cpu().numpy().T)
    return outs[0] + 1j * outs[1] if cplx else outs[0]


def hsrq3in_dense(a, eigenvalues, config=None, device=None):
    """Eigenvectors of a dense real A for the given eigenvalues of A:
    H, Q0 = householder_hessenberg(A); x = hsrq3in(H, ...); z = Q0 x.
    Returns the EigvecResult of hsrq3in with ``vectors`` replaced by z (unit
    2-norm, since Q0 is orthogonal) and ``hessenberg`` = (H, Q0)."""
    from .inviter import hsrq3in

    h, q = householder_hessenberg(a, device)
    res = hsrq3in(HessenbergMatrix(np.triu(h, -1)), eigenvalues, config)
    res.vectors = backmultiply(q, res.vectors, device)
    res.hessenberg = (h, q)
    return res


__all__ = ["householder_hessenberg", "hessenberg_device", "backmultiply", "backmultiply_device",
           "hsrq3in_dense"]
