"""The GPU seam: one call of libhsrq_b200 per solve group.

Replaces hessrq's ``_solve_group`` (inviter.py:91-106) and the engine of
``dhsrq3``/``chsrq3`` (backsolve.py:350-388).  PyTorch supplies device memory
and the stream; all arithmetic runs in the CUDA kernels of csrc/.  A solve
group may mix real and complex shifts: the kernels place complex shifts
first (two real columns each) and real shifts after (include/hsrq.h).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import (
    ConfigError,
    HessenbergMatrix,
    ScalingMatrix,
    SingularSystemError,
    SingularTaskError,
    SolutionBlock,
    StructuralTaskError,
    StructuralViolationError,
    task_node_of_failure,
)

MAX_TILE = 128  # b_r limit of the GPU path (one warp holds a tile column)
_KIND_DEGENERATE = 1
_KIND_SINGULAR = 2


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("the hsrq B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


HOST_CHECK_MAX_N = 2048  # structure check on the host up to this n (cheap), else on the device


class HostHessenberg:
    """The caller's array before upload, with the checks that need no device:
    shape / dtype (core.py:66-69), the structure check for n <= 2048
    (core.py:70-73; larger matrices are checked by hsrq_h_upload on the
    device, same boolean), and is_unreduced (core.py:86-91, the subdiagonal
    only).  No copy unless the dtype or the memory layout requires one."""

    def __init__(self, h):
        a = np.asarray(h)
        if a.dtype != np.float64:
            a = np.array(a, dtype=np.float64, order="F")
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ConfigError(f"expected a square matrix, got shape {a.shape}")
        if not (a.flags.c_contiguous or a.flags.f_contiguous):
            a = np.asfortranarray(a)
        n = a.shape[0]
        if 3 <= n <= HOST_CHECK_MAX_N:
            low = a[2:, :-2]
            if np.any(low[np.tril_indices(n - 2)] != 0.0):
                raise ConfigError("matrix has nonzeros below the first subdiagonal")
        self.a = a
        self.n = n
        self.unreduced = bool(n == 1 or np.all(a[np.arange(1, n), np.arange(0, n - 1)] != 0.0))

    def is_unreduced(self):
        return self.unreduced


class DeviceHessenberg:
    """H resident in HBM, column-major with an even leading dimension.

    ``norm_inf`` / ``unreduced`` are HessenbergMatrix.infinity_norm() /
    is_unreduced() (core.py:80-93), bit for bit."""

    def __init__(self, h, device=None):
        hm = h if isinstance(h, HessenbergMatrix) else HessenbergMatrix(h)
        self.n = hm.n
        self.device = device or default_device()
        self.ldh = self.n + (self.n & 1)
        self.t = torch.zeros((self.n, self.ldh), dtype=torch.float64, device=self.device)
        self._upload(hm.data)
        self.norm_inf = hm.infinity_norm()
        self.unreduced = hm.is_unreduced()

    def _upload(self, a):
        """hsrq_h_upload: pinned-ring staged copy (+ device transpose of a
        C-order array) and the structure / norm checks; returns the checks."""
        lib = _lib.load()
        order = 1 if a.flags.f_contiguous else 0
        chk = np.zeros(3)
        st = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            r = lib.hsrq_h_upload(ctypes.c_void_p(a.ctypes.data), order, self.n, _ptr(self.t),
                                  self.ldh, ctypes.c_void_p(chk.ctypes.data),
                                  ctypes.c_void_p(st.cuda_stream))
        if r < 0:
            raise RuntimeError(f"hsrq_h_upload failed ({r}): {_lib.last_error()}")
        return chk

    @classmethod
    def upload(cls, h, device=None):
        """Validate and upload a caller's array the way HessenbergMatrix(h)
        does (core.py:66-77: float64, square, zero below the subdiagonal --
        the same ConfigError messages), without the host-side F-order copy:
        the array goes to the device as it lies in memory and the structure
        check and the infinity norm (the reference's left-to-right row sums
        of its F-order copy) run on the device, exactly."""
        hv = h if isinstance(h, HostHessenberg) else HostHessenberg(h)
        a = hv.a
        self = cls.__new__(cls)
        self.n = a.shape[0]
        self.device = device or default_device()
        self.ldh = self.n + (self.n & 1)
        self.t = torch.empty((self.n, self.ldh), dtype=torch.float64, device=self.device)
        if self.ldh != self.n:
            self.t[:, self.n:].zero_()
        chk = self._upload(a)
        if self.n >= 3 and chk[1] != 0:
            raise ConfigError("matrix has nonzeros below the first subdiagonal")
        self.norm_inf = float(chk[0])
        self.unreduced = bool(self.n == 1 or chk[2] == 0)
        return self

    def infinity_norm(self):
        return self.norm_inf

    def is_unreduced(self):
        return self.unreduced

    @classmethod
    def of(cls, h, device=None):
        """Cached device copy attached to a HessenbergMatrix."""
        hm = h if isinstance(h, HessenbergMatrix) else HessenbergMatrix(h)
        dev = device or default_device()
        key = str(dev)
        d = hm._device.get(key)
        if d is None:
            d = cls(hm, dev)
            hm._device[key] = d
        return d


@dataclass
class GroupOutput:
    """Device-side results of one solve group (torch tensors)."""

    X: torch.Tensor          # (ncol, n): row c = column c
    c_re: torch.Tensor       # (ms, n); compact: Stewart code t (real) / t1 (complex)
    c_im: torch.Tensor       # (ms, n); compact: (mc, n) codes t2
    s: torch.Tensor          # (ms, n); compact: None
    seg_exp: torch.Tensor    # (N, ms) int32
    alpha_exp: torch.Tensor  # (ms,) int32
    norms: torch.Tensor
    log2norm: torch.Tensor
    fail: torch.Tensor       # (ms,) int64
    nfail: int
    mc: int
    mr: int
    launches: int
    compact: bool = False
    perm: np.ndarray | None = None  # complex shifts' run order (solve_group(unpermute=False))

    def rotations(self):
        """The recorded rotations as (c_re, c_im, s) device tensors (ms, n),
        decoded from the compact codes when stored compactly (hsrq_compact_decode)."""
        if not self.compact:
            return self.c_re, self.c_im, self.s
        lib = _lib.load()
        ms, n = self.c_re.shape
        cr, ci, s = (torch.zeros((ms, n), dtype=torch.float64, device=self.c_re.device)
                     for _ in range(3))
        st = ctypes.c_void_p(torch.cuda.current_stream(self.c_re.device).cuda_stream)
        if self.mc:
            lib.hsrq_compact_decode(self.mc * n, 1, _ptr(self.c_re), _ptr(self.c_im), _ptr(cr),
                                    _ptr(ci), _ptr(s), st)
        if self.mr:
            off = self.mc
            lib.hsrq_compact_decode(self.mr * n, 0, _ptr(self.c_re[off:]), None, _ptr(cr[off:]),
                                    None, _ptr(s[off:]), st)
        return cr, ci, s


def compact_encode(c_re, c_im, s):
    """GivensTable.compact() on device tensors (core.py:193-199): real tables
    (c_im None) -> t; complex -> (t1, t2).  Bit-identical to givens.py."""
    lib = _lib.load()
    st = ctypes.c_void_p(torch.cuda.current_stream(c_re.device).cuda_stream)
    c_re, s = c_re.contiguous(), s.contiguous()
    t1 = torch.empty_like(c_re)
    if c_im is None:
        lib.hsrq_compact_encode(c_re.numel(), 0, _ptr(c_re), None, _ptr(s), _ptr(t1), None, st)
        return t1
    c_im = c_im.contiguous()
    t2 = torch.empty_like(c_re)
    lib.hsrq_compact_encode(c_re.numel(), 1, _ptr(c_re), _ptr(c_im), _ptr(s), _ptr(t1), _ptr(t2), st)
    return t1, t2


def compact_decode(t1, t2=None):
    """GivensTable.from_compact() on device tensors (core.py:201-209):
    returns (c, s) for real codes, (c_re, c_im, s) for complex pairs."""
    lib = _lib.load()
    st = ctypes.c_void_p(torch.cuda.current_stream(t1.device).cuda_stream)
    t1 = t1.contiguous()
    c, s = torch.empty_like(t1), torch.empty_like(t1)
    if t2 is None:
        lib.hsrq_compact_decode(t1.numel(), 0, _ptr(t1), None, _ptr(c), None, _ptr(s), st)
        return c, s
    t2 = t2.contiguous()
    ci = torch.empty_like(t1)
    lib.hsrq_compact_decode(t1.numel(), 1, _ptr(t1), _ptr(t2), _ptr(c), _ptr(ci), _ptr(s), st)
    return c, ci, s


MODE_COMPACT_ROTATIONS = 0x10  # include/hsrq.h


class GroupSolver:
    """Device buffers for one (n, b_r, m_cplx, m_real) shape, reusable across calls."""

    def __init__(self, dh: DeviceHessenberg, b_r, m_cplx, m_real, compact=False):
        if not (1 <= b_r <= dh.n):
            raise ConfigError(f"tile size b_r={b_r} out of range for n={dh.n}")
        if b_r > MAX_TILE:
            raise ConfigError(f"the B200 path supports b_r <= {MAX_TILE} (got {b_r})")
        self.lib = _lib.load()
        self.dh = dh
        self.n, self.b_r = dh.n, int(b_r)
        self.N = (self.n + self.b_r - 1) // self.b_r
        self.mc, self.mr = int(m_cplx), int(m_real)
        self.ms = self.mc + self.mr
        self.ncol = 2 * self.mc + self.mr
        dev = dh.device
        f64 = dict(dtype=torch.float64, device=dev)
        self.X = torch.empty((self.ncol, self.n), **f64)
        self.compact = bool(compact)
        self.c_re = torch.empty((self.ms, self.n), **f64)
        if self.compact:  # Stewart codes: 1 real per real rotation, 2 per complex one
            self.c_im = torch.empty((max(self.mc, 1), self.n), **f64)
            self.s = None
        else:
            self.c_im = torch.empty((self.ms, self.n), **f64)
            self.s = torch.empty((self.ms, self.n), **f64)
        self.seg_exp = torch.empty((self.N, self.ms), dtype=torch.int32, device=dev)
        self.alpha_exp = torch.empty(self.ms, dtype=torch.int32, device=dev)
        self.norms = torch.empty(self.ms, **f64)
        self.log2norm = torch.empty(self.ms, **f64)
        self.fail = torch.empty(self.ms, dtype=torch.int64, device=dev)
        self.lam_re = torch.empty(self.ms, **f64)
        self.lam_im = torch.empty(self.ms, **f64)
        self.ws_bytes = int(self.lib.hsrq_workspace_bytes(self.n, self.b_r, self.mc, self.mr))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)

    def set_shifts(self, lam_cplx, lam_real):
        lam = np.concatenate([np.asarray(lam_cplx, dtype=np.complex128).ravel(),
                              np.asarray(lam_real, dtype=np.float64).ravel().astype(np.complex128)])
        self.lam_re.copy_(torch.from_numpy(np.ascontiguousarray(lam.real)))
        self.lam_im.copy_(torch.from_numpy(np.ascontiguousarray(lam.imag)))

    def launch(self, B, broadcast, robust=True, mode="eigvec", stream=None, sync=True,
               omega=None):
        """Enqueue the whole sweep.  B: device (n,) vector (broadcast) or (ncol, n).
        ``omega``: the caller's OverflowBudget.omega (default DBL_MAX/2/b_r)."""
        stream = stream or torch.cuda.current_stream(self.dh.device)
        mode_i = {"solve": 0, "eigvec": 1}[mode] | (MODE_COMPACT_ROTATIONS if self.compact else 0)
        args = (
            _ptr(self.dh.t), self.dh.ldh, self.n, self.b_r, _ptr(self.lam_re), _ptr(self.lam_im),
            self.mc, self.mr, _ptr(B), 0 if broadcast else self.n, 1 if broadcast else 0,
            _ptr(self.X), self.n, _ptr(self.c_re), _ptr(self.c_im), _ptr(self.s), self.n,
            _ptr(self.seg_exp), _ptr(self.alpha_exp), _ptr(self.norms), _ptr(self.log2norm),
            _ptr(self.fail), int(bool(robust)), mode_i, _ptr(self.ws), self.ws_bytes,
            ctypes.c_void_p(stream.cuda_stream),
        )
        if omega is not None:
            if not sync:
                raise ConfigError("a custom overflow budget needs a synchronous launch")
            r = self.lib.hsrq_solve_group_omega(*args[:24], float(omega), *args[24:])
        else:
            fn = self.lib.hsrq_solve_group if sync else self.lib.hsrq_solve_group_async
            r = fn(*args)
        if r < 0:
            raise RuntimeError(f"hsrq_solve_group failed ({r}): {_lib.last_error()}")
        return int(r)

    def capture(self, B, broadcast, robust=True, mode="eigvec", stream=None):
        """Capture this solve (all its kernels and stream forks) as a CUDA graph
        (hsrq_graph_capture).  ``B`` must stay alive: replays read it, and the
        shifts in ``lam_re`` / ``lam_im`` (``set_shifts``) as they are then."""
        stream = stream or torch.cuda.current_stream(self.dh.device)
        mode_i = {"solve": 0, "eigvec": 1}[mode] | (MODE_COMPACT_ROTATIONS if self.compact else 0)
        g = ctypes.c_void_p()
        r = self.lib.hsrq_graph_capture(
            _ptr(self.dh.t), self.dh.ldh, self.n, self.b_r, _ptr(self.lam_re), _ptr(self.lam_im),
            self.mc, self.mr, _ptr(B), 0 if broadcast else self.n, 1 if broadcast else 0,
            _ptr(self.X), self.n, _ptr(self.c_re), _ptr(self.c_im), _ptr(self.s), self.n,
            _ptr(self.seg_exp), _ptr(self.alpha_exp), _ptr(self.norms), _ptr(self.log2norm),
            _ptr(self.fail), int(bool(robust)), mode_i, _ptr(self.ws), self.ws_bytes,
            ctypes.c_void_p(stream.cuda_stream), ctypes.byref(g))
        if r < 0:
            raise RuntimeError(f"hsrq_graph_capture failed ({r}): {_lib.last_error()}")
        self.release_graph()
        self._graph = g
        self._graph_b = B
        return self

    def replay(self, stream=None, sync=True):
        """Replay the captured solve; returns the failure count when ``sync``."""
        stream = stream or torch.cuda.current_stream(self.dh.device)
        st = ctypes.c_void_p(stream.cuda_stream)
        if self.lib.hsrq_graph_launch(self._graph, st) < 0:
            raise RuntimeError(f"hsrq_graph_launch failed: {_lib.last_error()}")
        if sync:
            return int(self.lib.hsrq_failure_count(_ptr(self.ws), st))
        return None

    def release_graph(self):
        g = getattr(self, "_graph", None)
        if g is not None:
            self.lib.hsrq_graph_destroy(g)
            self._graph = None

    def __del__(self):
        try:
            self.release_graph()
        except Exception:  # interpreter shutdown
            pass

    def output(self, nfail):
        return GroupOutput(self.X, self.c_re, self.c_im, self.s, self.seg_exp, self.alpha_exp,
                           self.norms, self.log2norm, self.fail, nfail, self.mc, self.mr,
                           int(self.lib.hsrq_last_launch_count()), self.compact)


@dataclass
class HostOutput:
    """Host-side results of one solve group through hsrq_solve_group_host."""

    X: np.ndarray          # (ncol, n): row c = column c
    seg_exp: np.ndarray    # (N, ms) int32
    alpha_exp: np.ndarray  # (ms,) int32
    norms: np.ndarray
    log2norm: np.ndarray
    fail: np.ndarray       # (ms,) int64
    nfail: int
    mc: int
    mr: int


class HostGroupSolver:
    """hsrq_solve_group_host: host (numpy, ideally pinned) buffers in and out.

    The reference's own calling convention for the seam -- ``_solve_group``
    takes and returns numpy arrays (inviter.py:91-106); only the reusable
    device workspace is a device allocation.  H streams to the device in
    column blocks overlapped with the sweep (include/hsrq.h).
    """

    def __init__(self, n, b_r, m_cplx, m_real, device=None):
        if not (1 <= b_r <= n):
            raise ConfigError(f"tile size b_r={b_r} out of range for n={n}")
        if b_r > MAX_TILE:
            raise ConfigError(f"the B200 path supports b_r <= {MAX_TILE} (got {b_r})")
        self.lib = _lib.load()
        self.n, self.b_r, self.mc, self.mr = int(n), int(b_r), int(m_cplx), int(m_real)
        self.ms = self.mc + self.mr
        self.ncol = 2 * self.mc + self.mr
        self.N = (self.n + self.b_r - 1) // self.b_r
        self.device = device or default_device()
        self.ws_bytes = int(self.lib.hsrq_host_workspace_bytes(self.n, self.b_r, self.mc, self.mr))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)

    def launch(self, h, lam_re, lam_im, b, broadcast, out, robust=True, mode="eigvec",
               stream=None, wait=True):
        """h: (n, n) float64 column-major (Fortran) array; lam_*: (ms,) complex-first;
        b: (n,) start vector (broadcast) or (ncol, n) rows = columns; out: HostOutput.
        ``wait=False`` enqueues only (hsrq_solve_group_host_async) and returns the
        ticket for ``wait_ticket``; the host buffers must stay alive until then."""
        h = np.asarray(h)
        if not (h.flags.f_contiguous and h.dtype == np.float64):
            if not wait:  # a converted copy could be freed while the copy engine reads it
                raise ConfigError("asynchronous launch needs a float64 Fortran-ordered h")
            h = np.asfortranarray(h, dtype=np.float64)
        # the C ABI reads raw pointers: wrong dtypes / strides would be read silently
        for name, a, dt in (("lam_re", lam_re, np.float64), ("lam_im", lam_im, np.float64),
                            ("b", b, np.float64), ("out.X", out.X, np.float64),
                            ("out.seg_exp", out.seg_exp, np.int32),
                            ("out.alpha_exp", out.alpha_exp, np.int32),
                            ("out.norms", out.norms, np.float64),
                            ("out.log2norm", out.log2norm, np.float64),
                            ("out.fail", out.fail, np.int64)):
            if a is None and name == "lam_im":
                continue
            if not (isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous):
                raise ConfigError(f"{name} must be a C-contiguous {np.dtype(dt).name} array")
        if lam_re.size != self.ms or (lam_im is not None and lam_im.size != self.ms):
            raise ConfigError("shift arrays must hold m_cplx + m_real entries")
        if b.size != (self.n if broadcast else self.n * self.ncol) or out.X.size != self.n * self.ncol:
            raise ConfigError("right-hand side / output sizes do not match the solver's shape")
        stream = stream or torch.cuda.current_stream(self.device)
        P = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)
        mode_i = {"solve": 0, "eigvec": 1}[mode]
        fn = self.lib.hsrq_solve_group_host if wait else self.lib.hsrq_solve_group_host_async
        r = fn(
            P(h), h.shape[0], self.n, self.b_r, P(lam_re), P(lam_im), self.mc, self.mr, P(b),
            0 if broadcast else self.n, 1 if broadcast else 0, P(out.X), self.n, P(out.seg_exp),
            P(out.alpha_exp), P(out.norms), P(out.log2norm), P(out.fail), int(bool(robust)),
            mode_i, _ptr(self.ws), self.ws_bytes, ctypes.c_void_p(stream.cuda_stream))
        if r < 0:
            raise RuntimeError(f"hsrq_solve_group_host failed ({r}): {_lib.last_error()}")
        if not wait:
            return int(r)
        out.nfail = int(r)
        return out

    def wait_ticket(self, ticket, out):
        """Complete an asynchronous launch: outputs on the host, ``out.nfail`` set."""
        r = self.lib.hsrq_host_wait(int(ticket))
        if r < 0:
            raise RuntimeError(f"hsrq_host_wait failed ({r}): {_lib.last_error()}")
        out.nfail = int(r)
        return out

    def new_output(self, pinned=False):
        def alloc(shape, dtype):
            if pinned:
                return torch.empty(shape, dtype=dtype).pin_memory().numpy()
            return np.empty(shape, dtype=torch.empty(0, dtype=dtype).numpy().dtype)

        return HostOutput(X=alloc((self.ncol, self.n), torch.float64),
                          seg_exp=alloc((self.N, self.ms), torch.int32),
                          alpha_exp=alloc((self.ms,), torch.int32),
                          norms=alloc((self.ms,), torch.float64),
                          log2norm=alloc((self.ms,), torch.float64),
                          fail=alloc((self.ms,), torch.int64), nfail=0, mc=self.mc, mr=self.mr)


def solve_group_host(h, eigs_cplx, eigs_real, b, b_r, *, robust=True, mode="eigvec",
                     device=None):
    """One solve group through the host-buffer entry point; returns HostOutput."""
    hm = h if isinstance(h, HessenbergMatrix) else HessenbergMatrix(h)
    _check_h(hm)
    mc = len(np.atleast_1d(eigs_cplx)) if eigs_cplx is not None else 0
    mr = len(np.atleast_1d(eigs_real)) if eigs_real is not None else 0
    hs = HostGroupSolver(hm.n, b_r, mc, mr, device)
    lam = np.concatenate([np.asarray(eigs_cplx if mc else [], dtype=np.complex128).ravel(),
                          np.asarray(eigs_real if mr else [], dtype=np.float64).ravel()
                          .astype(np.complex128)])
    bb = np.ascontiguousarray(b, dtype=np.float64)
    broadcast = bb.ndim == 1
    if not broadcast and bb.shape == (hm.n, hs.ncol):
        bb = np.ascontiguousarray(bb.T)
    out = hs.new_output()
    return hs.launch(np.asfortranarray(hm.data), np.ascontiguousarray(lam.real),
                     np.ascontiguousarray(lam.imag), bb, broadcast, out, robust=robust, mode=mode)


def _check_h(hm):
    if not hm.is_unreduced():
        raise ConfigError("matrix must be unreduced (nonzero subdiagonal)")


def raise_first_failure(fail_codes, b_c, kinds, n_tiles=None):
    """Raise the exception the reference would raise first.

    ``fail_codes`` per shift of one solve call (inviter/backsolve call order),
    ``kinds`` a list of (start, stop) shift ranges, each one reference call
    (its own batches).  Reference order: every reduction precedes every solve
    (tiled_reduce runs before _substitute), batches in order, tile columns
    right to left, rows bottom-up within a kernel, then the batch-local shift
    (scheduler.py:189-219, numba_backend.py:79-106, 138-192).

    What is raised is what the reference's caller sees: the executor's
    ``TaskError`` (scheduler.py:182-187) naming the failing graph node, with
    the kernel's ``SingularSystemError`` / ``StructuralViolationError`` as its
    ``cause`` / ``__cause__`` -- as ``SingularTaskError`` /
    ``StructuralTaskError`` (core.py here), which are instances of both.
    ``n_tiles`` (the grid's N) gives the node its ``seq``.
    """
    codes = np.asarray(fail_codes, dtype=np.int64)
    best = None
    for call_i, (lo, hi) in enumerate(kinds):
        sub = codes[lo:hi]
        bad = np.nonzero(sub)[0]
        if bad.size == 0:
            continue
        for phase in (_KIND_DEGENERATE, _KIND_SINGULAR):
            cands = []
            for q in bad:
                code = int(sub[q])
                ph, tile, row = code >> 56, (code >> 24) & 0xFFFFFFFF, code & 0xFFFFFF
                if ph != phase:
                    continue
                bc = max(1, min(b_c, hi - lo))
                cands.append(((q // bc), -tile, -row, q % bc, q, tile, row))
            if cands:
                best = (phase,) + min(cands)
                break
        if best is not None:
            break
    if best is None:
        return
    phase, batch, _t, _r, _l, q, tile, row = best
    node = task_node_of_failure(phase == _KIND_SINGULAR, int(tile), int(batch), n_tiles)
    if phase == _KIND_DEGENERATE:
        cause = StructuralViolationError(
            f"degenerate rotation in tile column {tile} at local row {row}, "
            f"shift {q} (both pivot entries are zero)")
        raise StructuralTaskError(node, cause) from cause
    cause = SingularSystemError(
        f"singular triangular factor for shift {q} (local row {row})",
        shift_index=int(q), local_index=int(row))
    raise SingularTaskError(node, cause) from cause


def solve_group(h, eigs_cplx, eigs_real, b, b_r, *, robust=True, mode="eigvec", b_c=32,
                device=None, solver=None, compact=False, unpermute=True, omega=None):
    """Run one solve group; returns (GroupOutput, GroupSolver).

    ``h``: a HessenbergMatrix / array, or a DeviceHessenberg already on the
    device.  ``b``: a real n-vector used for every column (the
    inverse-iteration start vector) or a host/device matrix (n, ncol) in the
    column layout.  ``unpermute=False`` leaves the complex shifts in the
    order they ran (sorted by imaginary part) and returns that order in
    ``GroupOutput.perm`` (None: caller order), for callers that map columns
    themselves (the inverse-iteration drivers' output packing).
    """
    if isinstance(h, DeviceHessenberg):
        dh = h
        if not dh.is_unreduced():
            raise ConfigError("matrix must be unreduced (nonzero subdiagonal)")
    else:
        hm = h if isinstance(h, HessenbergMatrix) else HessenbergMatrix(h)
        _check_h(hm)
        dh = DeviceHessenberg.of(hm, device)
    mc = len(np.atleast_1d(eigs_cplx)) if eigs_cplx is not None else 0
    mr = len(np.atleast_1d(eigs_real)) if eigs_real is not None else 0
    gs = solver or GroupSolver(dh, b_r, mc, mr, compact=compact)
    ec = np.asarray(eigs_cplx if mc else [], dtype=np.complex128).ravel()
    # Complex shifts run sorted by imaginary part: the DP-lane sweep takes a
    # guard's exact pass when any shift of a warp needs it, and neighbouring
    # shifts then need it together more often (config 5: diag 135.8 -> 132.7
    # ms).  Columns are independent, so this changes no result; the outputs
    # are put back in the caller's order below.
    perm = np.argsort(ec.imag, kind="stable") if mc > 1 else None
    if perm is not None and np.array_equal(perm, np.arange(mc)):
        perm = None
    gs.set_shifts(ec[perm] if perm is not None else ec, eigs_real if mr else [])
    bt = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64))
    broadcast = bt.dim() == 1
    if not broadcast:
        bt = bt.T.contiguous() if bt.shape[0] == hm.n and bt.shape[1] == gs.ncol else bt
    bt = bt.to(dh.device)
    if perm is not None and not broadcast:  # right-hand sides follow their shifts
        bt = bt[torch.from_numpy(_col_index(perm, mc, mr)).to(bt.device)].contiguous()
    nfail = gs.launch(bt, broadcast, robust=robust, mode=mode, omega=omega)
    if perm is not None and unpermute:
        _unpermute(gs, perm)
        perm = None
    out = gs.output(nfail)
    out.perm = perm
    return out, gs


def _col_index(perm, mc, mr):
    """Real-column index map of a complex-shift permutation (complex shift q
    owns columns 2q, 2q+1; real columns follow unchanged)."""
    cols = np.empty(2 * mc, dtype=np.int64)
    cols[0::2] = 2 * perm
    cols[1::2] = 2 * perm + 1
    return np.concatenate([cols, 2 * mc + np.arange(mr, dtype=np.int64)])


def _unpermute(gs, perm):
    """Outputs of a solve run with complex shifts in order ``perm`` back to the
    caller's order (device copies; rows / columns of every per-shift array)."""
    dev = gs.X.device
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    qi = torch.from_numpy(np.concatenate([inv, perm.size + np.arange(gs.mr)])).to(dev)
    ci = torch.from_numpy(_col_index(inv, gs.mc, gs.mr)).to(dev)
    gs.X.copy_(gs.X[ci])
    for t in (gs.c_re, gs.s):
        if t is not None:
            t.copy_(t[qi])
    if gs.compact:
        gs.c_im[: gs.mc].copy_(gs.c_im[: gs.mc][torch.from_numpy(inv).to(dev)])
    else:
        gs.c_im.copy_(gs.c_im[qi])
    gs.seg_exp.copy_(gs.seg_exp[:, qi])
    for t in (gs.alpha_exp, gs.norms, gs.log2norm, gs.fail):
        t.copy_(t[qi])
    gs.lam_re.copy_(gs.lam_re[qi])
    gs.lam_im.copy_(gs.lam_im[qi])


def to_solution_block(out: GroupOutput, n, *, robust=True, want_cplx):
    """Host SolutionBlock in the reference's layout for a single-kind group."""
    X = out.X.cpu().numpy()
    if want_cplx:
        x = (X[0 : 2 * out.mc : 2] + 1j * X[1 : 2 * out.mc : 2]).T.copy()
    else:
        x = X[2 * out.mc :].T.copy()
    sl = slice(0, out.mc) if want_cplx else slice(out.mc, out.mc + out.mr)
    seg = out.seg_exp.cpu().numpy()[:, sl].copy()
    aexp = out.alpha_exp.cpu().numpy()[sl].copy()
    norms = out.norms.cpu().numpy()[sl].copy()
    l2 = out.log2norm.cpu().numpy()[sl].copy()
    if not robust:
        return SolutionBlock(x=x, alpha=np.ones(aexp.size),
                             segment_scales=ScalingMatrix(np.ones(seg.shape), np.zeros_like(seg)),
                             norms=None, alpha_exp=np.zeros_like(aexp))
    return SolutionBlock(x=x, alpha=np.ldexp(1.0, aexp),
                         segment_scales=ScalingMatrix(np.ldexp(1.0, seg), seg), norms=norms,
                         alpha_exp=aexp, log2_norms=l2)


def converged_log2(log2_norm, n):
    """``converged`` (inviter.py:71-73) evaluated on log2 of the represented norm."""
    return log2_norm > math.log2(0.1 / math.sqrt(n))
