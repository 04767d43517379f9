"""Types and errors of the reference's solver surface (hessrq core.py), as
the B200 path consumes and returns them.

Only what the inverse-iteration seam needs: the matrix wrapper (core.py:60-102),
the tile grid (:105-129), the scaling matrix / solution block (:234-260) and
the error hierarchy (:39-57), with the same names and semantics so existing
callers catch the same exceptions.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class HessrqError(Exception):
    """Base class for numerical / structural failures (core.py:39-40)."""


class ConfigError(HessrqError):
    """Invalid configuration (core.py:43-44)."""


class SingularSystemError(HessrqError):
    """An exactly singular triangular factor was met (core.py:47-53)."""

    def __init__(self, message, shift_index=None, local_index=None):
        super().__init__(message)
        self.shift_index = shift_index
        self.local_index = local_index


class StructuralViolationError(HessrqError):
    """Input violates the unreduced-Hessenberg structure (core.py:56-57)."""


@dataclass
class TaskNode:
    """The reference's task-graph node (scheduler.py:35-43) as far as a failure
    report needs it: ``kind`` ("ReduceDiag", "SolveTile",
    "MergedSolveBacktransform"), ``coords`` = (tile_i, tile_j, batch) and the
    node's position ``seq`` in the reference's graph (scheduler.py:120-179)."""

    kind: str
    coords: tuple
    seq: int = None
    run: object = None

    def __repr__(self):
        return f"TaskNode({self.kind}, coords={self.coords})"


class TaskError(Exception):
    """What a caller of the reference actually catches when a kernel fails: the
    executor aborts the graph and re-raises the kernel's error wrapped with the
    failing node (scheduler.py:182-187, 211-214) -- ``node``, ``cause``, the
    message ``task <kind> at <coords> failed: <cause>``, ``__cause__`` set."""

    def __init__(self, node, cause):
        Exception.__init__(self, f"task {node.kind} at {node.coords} failed: {cause}")
        self.node = node
        self.cause = cause


class SingularTaskError(TaskError, SingularSystemError):
    """The TaskError of a singular pivot.  It is also a SingularSystemError
    (``shift_index`` / ``local_index`` of the cause), so both ``except
    TaskError`` written against the reference's drivers and ``except
    SingularSystemError`` written against its kernels' error type catch it."""

    def __init__(self, node, cause):
        TaskError.__init__(self, node, cause)
        self.shift_index = cause.shift_index
        self.local_index = cause.local_index


class StructuralTaskError(TaskError, StructuralViolationError):
    """The TaskError of a degenerate rotation; also a StructuralViolationError."""


def task_node_of_failure(phase_singular, tile, batch, n_tiles):
    """The reference graph node in which a kernel failure surfaces: a degenerate
    rotation in ReduceDiag (tile, tile, batch) of the reduction graph, a singular
    pivot in SolveTile (tile, tile, batch) -- MergedSolveBacktransform (0, 0,
    batch) for tile 0 -- of the substitution graph; ``seq`` by the graphs'
    construction order (scheduler.py:120-179: batches outermost, tile columns
    right to left, the diagonal node first, then one node per tile row)."""
    N = n_tiles
    seq = None
    if N is not None:
        before = sum(1 + t for t in range(tile + 1, N))  # nodes of the columns to the right
        if phase_singular:
            per_batch = sum(1 + t for t in range(1, N)) + 1
            seq = batch * per_batch + (before if tile > 0 else per_batch - 1)
        else:
            per_batch = sum(1 + t for t in range(N))
            seq = batch * per_batch + before
    if not phase_singular:
        return TaskNode("ReduceDiag", (tile, tile, batch), seq)
    if tile == 0:
        return TaskNode("MergedSolveBacktransform", (0, 0, batch), seq)
    return TaskNode("SolveTile", (tile, tile, batch), seq)


class HessenbergMatrix:
    """Read-only real upper Hessenberg matrix (core.py:60-98 semantics)."""

    def __init__(self, data):
        a = np.array(data, dtype=np.float64, order="F")
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ConfigError(f"expected a square matrix, got shape {a.shape}")
        n = a.shape[0]
        if n >= 3 and np.any(np.tril(a, -2) != 0.0):
            raise ConfigError("matrix has nonzeros below the first subdiagonal")
        a.setflags(write=False)
        self.n = n
        self.data = a
        self._norm_inf = None
        self._device = {}

    def infinity_norm(self):
        if self._norm_inf is None:
            self._norm_inf = float(np.max(np.sum(np.abs(self.data), axis=1)))
        return self._norm_inf

    def is_unreduced(self):
        if self.n == 1:
            return True
        return bool(np.all(np.diagonal(self.data, -1) != 0.0))

    def subdiagonal(self):
        return np.diagonal(self.data, -1).copy()

    def __repr__(self):
        return f"HessenbergMatrix(n={self.n})"


def as_hessenberg(h):
    return h if isinstance(h, HessenbergMatrix) else HessenbergMatrix(h)


class TileGrid:
    """Row/column partition into b_r tiles, last one possibly short (core.py:105-129)."""

    def __init__(self, n, b_r):
        if not (1 <= b_r <= n):
            raise ConfigError(f"tile size b_r={b_r} out of range for n={n}")
        self.n = n
        self.b_r = b_r
        self.ranges = [(s, min(s + b_r, n)) for s in range(0, n, b_r)]
        self.N = len(self.ranges)

    def tile_of(self, i):
        return i // self.b_r

    def tile_slice(self, t):
        s, e = self.ranges[t]
        return slice(s, e)

    def __repr__(self):
        return f"TileGrid(n={self.n}, b_r={self.b_r}, N={self.N})"

    @property
    def tile_ends(self):
        return np.array([e for _s, e in self.ranges], dtype=np.int64)


_DBL_MAX = float(np.finfo(np.float64).max)


@dataclass(frozen=True)
class OverflowBudget:
    """The working overflow threshold omega (overflow.py:30-47): the ``budget=``
    argument of dhsrq3 / chsrq3.  Default: the true overflow limit over two and
    over the tile height."""

    omega: float
    safety_divisor: int = 1

    def __post_init__(self):
        if not (0.0 < self.omega <= _DBL_MAX / 2.0):
            raise ValueError(f"omega={self.omega} outside (0, maxfloat/2]")
        if self.omega * self.safety_divisor > _DBL_MAX:
            raise ValueError("omega * safety_divisor exceeds the representable range")

    @classmethod
    def for_tile_rows(cls, b_r):
        return cls(omega=_DBL_MAX / 2.0 / b_r, safety_divisor=int(b_r))

    @classmethod
    def for_grid(cls, grid):
        return cls.for_tile_rows(grid.b_r)


class Workspace:
    """The ``workspace=`` argument of the drivers (core.py:263-283): host scratch
    keyed by role, and the high-water mark of cross-over storage in reals.  The
    GPU path keeps its cross-over block on the device (O(n cols));
    ``peak_crossover_reals`` reports the reference's figure, n N cols, so caps
    written against the reference keep their meaning."""

    def __init__(self):
        self._bufs = {}
        self.peak_crossover_reals = 0

    def take(self, key, shape, dtype=np.float64, crossover=False):
        size = int(np.prod(shape))
        buf = self._bufs.get(key)
        if buf is None or buf.size < size or buf.dtype != np.dtype(dtype):
            buf = np.empty(size, dtype=dtype)
            self._bufs[key] = buf
        if crossover:
            self.peak_crossover_reals = max(self.peak_crossover_reals, size)
        return buf[:size].reshape(shape)


@dataclass
class ScalingMatrix:
    """Segment scales alpha(tile, shift) = 2**exponent (core.py:234-248)."""

    alpha: np.ndarray
    exponent: np.ndarray | None = None

    def __post_init__(self):
        self.alpha = np.asarray(self.alpha, dtype=np.float64)

    def all_ones(self):
        return bool(np.all(self.alpha == 1.0))


@dataclass
class SolutionBlock:
    """Solutions plus per-column scales and represented norms (core.py:251-260).

    Extra fields of the B200 path: ``alpha_exp`` / ``log2_norms`` keep the
    exact exponent and the log2 norm where the reference's doubles would
    underflow to 0 or overflow to inf.
    """

    x: np.ndarray
    alpha: np.ndarray
    segment_scales: ScalingMatrix | None = None
    norms: np.ndarray | None = None
    converged: np.ndarray | None = None
    flops: dict = field(default_factory=dict)
    alpha_exp: np.ndarray | None = None
    log2_norms: np.ndarray | None = None


def interleave_complex(z):
    """(n, m) complex -> (n, 2m) float with re/im in adjacent columns (core.py:286-292)."""
    z = np.asarray(z, dtype=np.complex128)
    out = np.empty((z.shape[0], 2 * z.shape[1]), dtype=np.float64)
    out[:, 0::2] = z.real
    out[:, 1::2] = z.imag
    return out


def deinterleave_complex(x):
    """(n, 2m) float interleaved -> (n, m) complex (core.py:295-300)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[1] % 2:
        raise ConfigError("interleaved array must have an even column count")
    return x[:, 0::2] + 1j * x[:, 1::2]


class RunStats:
    """Per-task-type time and flop accumulators (scheduler.py:98-119): the
    ``stats`` argument of dhsrq3 / chsrq3.  The B200 kernels fuse task types,
    so a solve adds each type once, with the measured fused-kernel time split
    in proportion to the reference flop model (see benchcsv.task_seconds)."""

    def __init__(self):
        self.seconds = {}
        self.flops = {}
        self.formula = {}
        self.calls = {}

    def add(self, task_type, seconds, flops=0.0, formula=0.0):
        self.seconds[task_type] = self.seconds.get(task_type, 0.0) + seconds
        self.flops[task_type] = self.flops.get(task_type, 0.0) + flops
        self.formula[task_type] = self.formula.get(task_type, 0.0) + formula
        self.calls[task_type] = self.calls.get(task_type, 0) + 1
