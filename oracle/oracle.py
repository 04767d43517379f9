"""ctypes front end of the CPU oracle (``hsrq_oracle.c``).

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline and ``--impl reference``) as the checker /
CPU baseline; the product package never imports it.

Layouts follow the reference: H column-major n x n; per-shift arrays are
C-order ``(n, m)`` (real) or interleaved ``(n, 2m)`` (complex), exactly what
``_substitute`` hands its kernels (backsolve.py:71-74).  Scale factors come
back both as int exponents (exact) and as the reference's doubles
``ldexp(1, e)``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libhsrq_oracle.so")
_lib = None

_EPS = float(np.finfo(np.float64).eps)
_DMAX = float(np.finfo(np.float64).max)

_d = ctypes.POINTER(ctypes.c_double)
_i32 = ctypes.POINTER(ctypes.c_int)
_i64 = ctypes.POINTER(ctypes.c_int64)


def build(force=False):
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "hsrq_oracle.c"))
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_hsrq_solve.restype = ctypes.c_int64
        L.oracle_hsrq_solve.argtypes = [
            _d, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
            _d, _d, _d, _d, _d, _d, _d, _i32, _i32, _d, _d, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, _i64,
        ]
        L.oracle_protect_update.restype = ctypes.c_double
        L.oracle_protect_update.argtypes = [ctypes.c_double] * 4
        L.oracle_pow2floor.restype = ctypes.c_double
        L.oracle_pow2floor.argtypes = [ctypes.c_double]
        L.oracle_set_blas.restype = None
        L.oracle_set_blas.argtypes = [ctypes.c_void_p] * 3
        for name in ("oracle_reduce_diag", "oracle_solve_rsolve", "oracle_creduce_diag",
                     "oracle_csolve_crsolve"):
            getattr(L, name).restype = ctypes.c_int64
        _lib = L
    return _lib


def reference_blas_pointer(name):
    """Address of the Fortran BLAS routine numba's np.dot binds (scipy.linalg.cython_blas)."""
    try:
        from scipy.linalg import cython_blas
    except Exception:  # pragma: no cover - scipy is in the image
        return None
    cap = cython_blas.__pyx_capi__[name]
    get_name = ctypes.pythonapi.PyCapsule_GetName
    get_name.restype = ctypes.c_char_p
    get_name.argtypes = [ctypes.py_object]
    get_ptr = ctypes.pythonapi.PyCapsule_GetPointer
    get_ptr.restype = ctypes.c_void_p
    get_ptr.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return get_ptr(cap, get_name(cap))


def use_reference_blas(enable=True):
    """Route the update GEMM through the reference's BLAS (bit-identical driver)."""
    if enable:
        lib().oracle_set_blas(*(reference_blas_pointer(f) for f in ("dgemm", "dgemv", "ddot")))
    else:
        lib().oracle_set_blas(None, None, None)


def blas_corename():
    """OpenBLAS kernel family scipy's BLAS dispatched to (fixes dgemm rounding)."""
    try:
        import glob
        import scipy

        libs = glob.glob(os.path.join(os.path.dirname(scipy.__file__) + ".libs", "libscipy_openblas*.so"))
        L = ctypes.CDLL(libs[0])
        for sym in ("scipy_openblas_get_corename", "openblas_get_corename"):
            if hasattr(L, sym):
                f = getattr(L, sym)
                f.restype = ctypes.c_char_p
                return f().decode()
    except Exception:
        pass
    return "unknown"


def _p(a, t=_d):
    return a.ctypes.data_as(t) if a is not None else None


def omega_for(b_r):
    """OverflowBudget.for_tile_rows (overflow.py:41-43)."""
    return _DMAX / 2.0 / b_r


def protect_update(bnorm, hnorm, xnorm, omega):
    return lib().oracle_protect_update(bnorm, hnorm, xnorm, omega)


def pow2floor(x):
    return lib().oracle_pow2floor(x)


@dataclass
class OracleResult:
    x: np.ndarray  # (n, m) float64 or complex128
    alpha: np.ndarray  # (m,) reference doubles ldexp(1, e)
    alpha_exp: np.ndarray  # (m,) int32
    segment_exp: np.ndarray  # (N, m) int32
    norms: np.ndarray  # (m,)
    log2norm: np.ndarray  # (m,)
    c_re: np.ndarray
    c_im: np.ndarray | None
    s: np.ndarray

    @property
    def segment_scales(self):
        return np.ldexp(1.0, self.segment_exp)


class OracleError(RuntimeError):
    def __init__(self, status, phase, tile, shift, row):
        kind = "degenerate rotation" if phase == 1 else "singular factor"
        super().__init__(f"{kind}: tile {tile}, shift {shift}, local row {row}")
        self.status, self.phase, self.tile, self.shift_index, self.local_index = (
            status, phase, tile, shift, row)


def solve(h, shifts, b, b_r, b_c=32, robust=True, mode="eigvec", nthreads=1):
    """dhsrq3/chsrq3 (+ _solve_group when mode='eigvec') on the CPU oracle.

    ``shifts`` real -> real solve; complex dtype -> complex solve (b complex).
    """
    L = lib()
    H = np.asfortranarray(np.asarray(h, dtype=np.float64))
    n = H.shape[0]
    lam = np.asarray(shifts).ravel()
    cplx = np.iscomplexobj(lam)
    m = lam.size
    N = (n + b_r - 1) // b_r
    lre = np.ascontiguousarray(lam.real, dtype=np.float64)
    lim = np.ascontiguousarray(lam.imag, dtype=np.float64) if cplx else None
    if cplx:
        bc = np.asarray(b, dtype=np.complex128).reshape(n, m)
        B = np.empty((n, 2 * m))
        B[:, 0::2] = bc.real
        B[:, 1::2] = bc.imag
    else:
        B = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n, m))
    X = np.empty_like(B)
    c_re = np.empty((n, m))
    c_im = np.empty((n, m)) if cplx else None
    s = np.empty((n, m))
    seg = np.zeros((N, m), dtype=np.int32)
    acol = np.zeros(m, dtype=np.int32)
    norms = np.empty(m)
    l2 = np.empty(m)
    err = np.zeros(4, dtype=np.int64)
    mode_i = {"solve": 0, "eigvec": 1}[mode]
    st = L.oracle_hsrq_solve(
        _p(H), n, int(b_r), int(min(b_c, m)), int(cplx), m, _p(lre), _p(lim), _p(B), _p(X),
        _p(c_re), _p(c_im), _p(s), _p(seg, _i32), _p(acol, _i32), _p(norms), _p(l2),
        int(robust), mode_i, int(nthreads), _p(err, _i64))
    if st != 0:
        raise OracleError(st, int(err[0]), int(err[1]), int(err[2]), int(err[3]))
    x = X[:, 0::2] + 1j * X[:, 1::2] if cplx else X
    return OracleResult(x=x, alpha=np.ldexp(1.0, acol), alpha_exp=acol, segment_exp=seg,
                        norms=norms, log2norm=l2, c_re=c_re, c_im=c_im, s=s)


# ---------------------------------------------------------------------------
# tile kernels (reference operator API, K/__init__.py), for tile-level parity
# ---------------------------------------------------------------------------

def reduce_diag(hdiag, hleft, has_left, lam, rright):
    hdiag = np.ascontiguousarray(hdiag, dtype=np.float64)
    rr = np.ascontiguousarray(rright, dtype=np.float64)
    k, b = rr.shape
    hl = np.ascontiguousarray(hleft, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    c = np.empty((k, b))
    s = np.empty((k, b))
    st = lib().oracle_reduce_diag(k, b, _p(hdiag), _p(hl), int(has_left), _p(lam), _p(rr), _p(c), _p(s))
    return st, c, s


def solve_rsolve(hdiag, hleft, has_left, lam, rright, c, s, x, beta_e, robust, omega):
    hdiag = np.ascontiguousarray(hdiag, dtype=np.float64)
    rr = np.ascontiguousarray(rright, dtype=np.float64)
    k, b = rr.shape
    args = [np.ascontiguousarray(a, dtype=np.float64) for a in (hleft, lam, c, s)]
    x = np.array(x, dtype=np.float64, order="C")
    be = np.array(beta_e, dtype=np.int32)
    st = lib().oracle_solve_rsolve(
        k, b, _p(hdiag), _p(args[0]), int(has_left), _p(args[1]), _p(rr), _p(args[2]),
        _p(args[3]), _p(x), _p(be, _i32), int(robust), ctypes.c_double(omega))
    return st, x, be


def creduce_diag(hdiag, hleft, has_left, lam_re, lam_im, rright2):
    hdiag = np.ascontiguousarray(hdiag, dtype=np.float64)
    rr = np.ascontiguousarray(rright2, dtype=np.float64)
    k = rr.shape[0]
    b = rr.shape[1] // 2
    hl = np.ascontiguousarray(hleft, dtype=np.float64)
    lre = np.ascontiguousarray(lam_re, dtype=np.float64)
    lim = np.ascontiguousarray(lam_im, dtype=np.float64)
    cre, cim, s = np.empty((k, b)), np.empty((k, b)), np.empty((k, b))
    st = lib().oracle_creduce_diag(k, b, _p(hdiag), _p(hl), int(has_left), _p(lre), _p(lim),
                                   _p(rr), _p(cre), _p(cim), _p(s))
    return st, cre, cim, s


def csolve_crsolve(hdiag, hleft, has_left, lam_re, lam_im, rright2, cre, cim, s, x2, beta_e,
                   robust, omega):
    hdiag = np.ascontiguousarray(hdiag, dtype=np.float64)
    rr = np.ascontiguousarray(rright2, dtype=np.float64)
    k = rr.shape[0]
    b = rr.shape[1] // 2
    args = [np.ascontiguousarray(a, dtype=np.float64) for a in (hleft, lam_re, lam_im, cre, cim, s)]
    x2 = np.array(x2, dtype=np.float64, order="C")
    be = np.array(beta_e, dtype=np.int32)
    st = lib().oracle_csolve_crsolve(
        k, b, _p(hdiag), _p(args[0]), int(has_left), _p(args[1]), _p(args[2]), _p(rr),
        _p(args[3]), _p(args[4]), _p(args[5]), _p(x2), _p(be, _i32), int(robust),
        ctypes.c_double(omega))
    return st, x2, be


def henry_solve(h, lam, b):
    """Henry's single sweep (henry_solve_real / henry_solve_complex,
    K/numba_backend.py:830-923) on an (n, m) right-hand side.

    Returns (status, x): the reference's packed status of the first failure
    (0 = ok) and x (n, m), float64 for real shifts, complex128 for complex."""
    L = lib()
    h = np.asfortranarray(h, dtype=np.float64)
    n = h.shape[0]
    lam = np.atleast_1d(np.asarray(lam))
    m = lam.shape[0]
    if np.iscomplexobj(lam):
        x = np.ascontiguousarray(np.asarray(b, dtype=np.complex128).reshape(n, m)).copy()
        lm = np.ascontiguousarray(lam, dtype=np.complex128)
        f = L.oracle_henry_solve_complex
    else:
        x = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n, m)).copy()
        lm = np.ascontiguousarray(lam, dtype=np.float64)
        f = L.oracle_henry_solve_real
    f.restype = ctypes.c_int64
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    st = int(f(h.ctypes.data, n, m, lm.ctypes.data, x.ctypes.data))
    return st, x


def compact_encode(c_re, s, c_im=None):
    """givens.compact_encode_table / _complex: t (real) or (t1, t2) (complex)."""
    L = lib()
    c_re = np.ascontiguousarray(c_re, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    t1 = np.empty_like(c_re)
    L.oracle_compact_encode.restype = None
    if c_im is None:
        L.oracle_compact_encode(ctypes.c_int64(c_re.size), 0, _p(c_re), None, _p(s), _p(t1), None)
        return t1
    c_im = np.ascontiguousarray(c_im, dtype=np.float64)
    t2 = np.empty_like(c_re)
    L.oracle_compact_encode(ctypes.c_int64(c_re.size), 1, _p(c_re), _p(c_im), _p(s), _p(t1), _p(t2))
    return t1, t2


def compact_decode(t1, t2=None):
    """givens.compact_decode_table / _complex: (c, s) or (c_re, c_im, s)."""
    L = lib()
    t1 = np.ascontiguousarray(t1, dtype=np.float64)
    c, s = np.empty_like(t1), np.empty_like(t1)
    L.oracle_compact_decode.restype = None
    if t2 is None:
        L.oracle_compact_decode(ctypes.c_int64(t1.size), 0, _p(t1), None, _p(c), None, _p(s))
        return c, s
    t2 = np.ascontiguousarray(t2, dtype=np.float64)
    ci = np.empty_like(t1)
    L.oracle_compact_decode(ctypes.c_int64(t1.size), 1, _p(t1), _p(t2), _p(c), _p(ci), _p(s))
    return c, ci, s


def householder_hessenberg(a):
    """testprob.householder_hessenberg restated (unblocked, C): returns (H, Q)."""
    L = lib()
    h = np.array(a, dtype=np.float64, order="F")
    n = h.shape[0]
    q = np.empty((n, n), order="F")
    L.oracle_householder_hessenberg.restype = None
    L.oracle_householder_hessenberg(ctypes.c_int64(n), _p(h), _p(q))
    return h, q


def set_omega(omega):
    """Test hook: solves use OverflowBudget(omega) (0 / None: DBL_MAX/2/b_r)."""
    L = lib()
    L.oracle_set_omega.restype = None
    L.oracle_set_omega.argtypes = [ctypes.c_double]
    L.oracle_set_omega(float(omega or 0.0))


def set_stop(jt):
    """Test hook: oracle solves end after tile column jt's updates (no
    backtransform; x holds solved tiles >= jt and updated rhs below); -1 off."""
    L = lib()
    L.oracle_set_stop.restype = None
    L.oracle_set_stop.argtypes = [ctypes.c_int]
    L.oracle_set_stop(int(jt))
