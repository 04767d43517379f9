"""Multi-GPU inverse iteration: shifts partitioned, H replicated, X gathered.

Every column of the solve is independent (no kernel couples shifts, and the
restart vectors depend only on the attempt index, inviter.py:76-88), so the
selection shards across ranks with no collective inside the sweep
(SURVEY.md §8(e)).  Per restart attempt the ranks exchange only a few bytes
(whether any shift is left anywhere, and the failure codes, so every rank
raises the reference's first failure, inviter.py:109-152 / backsolve.py:53-59);
at the end ONE point-to-point gather moves each rank's solution block to the
destination rank on the device -- real columns as one n-vector, complex
shifts as a re/im pair, exactly the bytes of X once (NCCL over NVLink on
B200, gloo on CPU in the tests) -- and the destination assembles the
caller-order result on its GPU (hsrq_pack_download).

Any exception on one rank (a CUDA error, a failed allocation) is announced to
the others at the next exchange, so every rank raises instead of the others
waiting forever in a collective.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .core import HessrqError

# flop-model ratio of a complex to a real shift at n=16000, b_r=128
# (1.3330e9 / 6.5329e8, hessrq flops.py)
COMPLEX_COST = 2.04


class ShardError(RuntimeError):
    """Another rank (or this one) failed outside the solver's own error path."""


def shard_bounds(n_real, n_cplx, world):
    """Per-kind shard boundaries: ``(real_cuts, cplx_cuts)``, each ``world + 1`` long.

    Every rank gets an equal share (to one shift) of the real AND of the
    complex shifts, so the flop cost (complex ~2.04 x real at n=16000) and the
    latency-bound diagonal sweeps of both kinds are balanced at once.
    """
    rc = np.array([(n_real * r) // world for r in range(world + 1)], dtype=np.int64)
    cc = np.array([(n_cplx * r) // world for r in range(world + 1)], dtype=np.int64)
    return rc, cc


def local_selection(eigenvalues, rank, world):
    """This rank's shifts (original indices, values) of a mixed selection:
    every world-th shift of each kind, in the order sorted by imaginary part
    -- the same counts as ``shard_bounds`` gives, but each rank a
    representative sample (the guard work of the diagonal sweeps varies along
    the spectrum, and the slowest rank sets the step time)."""
    eigs = np.asarray(eigenvalues, dtype=np.complex128).ravel()
    is_cplx = eigs.imag != 0.0
    ridx = np.nonzero(~is_cplx)[0]
    cidx = np.nonzero(is_cplx)[0]
    cidx = cidx[np.argsort(eigs[cidx].imag, kind="stable")]
    idx = np.concatenate([ridx[rank::world], cidx[rank::world]])
    return idx, eigs[idx]


class ShardExchange:
    """The per-attempt exchange of a sharded _iterate (inviter._iterate_mixed).

    Every rank performs the same sequence of collectives (one per
    ``any_remaining``, ``failures``, ``collect``), each carrying an error
    slot; ``poison`` fills it from a local exception, and whoever sees a
    filled slot raises ShardError.  ``r_glob`` / ``c_glob`` map this rank's
    local real / complex shift index to its position in the reference's
    dhsrq3in / chsrq3in call (real-first stable order, inviter.py:203-206).
    """

    def __init__(self, group, r_glob, c_glob):
        self.group = group
        self.r_glob = np.asarray(r_glob, dtype=np.int64)
        self.c_glob = np.asarray(c_glob, dtype=np.int64)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.calls = 0

    def _collect(self, payload, err=None):
        self.calls += 1
        out = [None] * self.world
        dist.all_gather_object(out, (err, payload), group=self.group)
        bad = [(r, e) for r, (e, _) in enumerate(out) if e is not None]
        if bad:
            raise ShardError("; ".join(f"rank {r}: {e}" for r, e in bad))
        return [p for _, p in out]

    def poison(self, exc):
        """Announce a local failure at the next collective (raises ShardError)."""
        self._collect(None, err=f"{type(exc).__name__}: {exc}")

    def any_remaining(self, count):
        return sum(self._collect(int(count))) > 0

    def failures(self, attempt, fr, rr, fc, rc, b_c, n_tiles=None):
        """All ranks' failure codes of this attempt, placed at their position
        in the reference's remaining-shift order; raises the first failure
        (solver.raise_first_failure) on every rank alike."""
        from .solver import raise_first_failure

        fr = np.asarray(fr, dtype=np.int64)
        fc = np.asarray(fc, dtype=np.int64)
        mine = (self.r_glob[rr].tolist(), fr.tolist(), self.c_glob[rc].tolist(), fc.tolist())
        alls = self._collect(mine)
        if not any(any(x[1]) or any(x[3]) for x in alls):
            return
        R = sorted((g, c) for x in alls for g, c in zip(x[0], x[1]))
        C = sorted((g, c) for x in alls for g, c in zip(x[2], x[3]))
        codes = np.array([c for _, c in R] + [c for _, c in C], dtype=np.int64)
        raise_first_failure(codes, b_c, [(0, len(R)), (len(R), len(R) + len(C))], n_tiles=n_tiles)

    def collect(self, payload):
        return self._collect(payload)


def gather_columns(X_local, counts, group=None, dst=0, out=None):
    """Point-to-point gather of every rank's solution block to ``dst``.

    ``X_local`` (ncol_r, n) on this rank's device (row c = column c; a real
    shift's column once, a complex shift's re/im pair); ``counts`` the ncol of
    every rank.  On ``dst`` returns the (sum ncol, n) block with rank r's rows
    at offset sum(counts[:r]) (``out`` if given); elsewhere None.  Exactly
    X's bytes cross the fabric once, no padding (NCCL send/recv on B200)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    n = X_local.shape[1] if X_local is not None and X_local.dim() == 2 else None
    if rank == dst:
        if n is None:
            raise ValueError("destination rank needs its (possibly empty) (ncol, n) block")
        Xall = out if out is not None else torch.empty((int(offs[-1]), n), dtype=X_local.dtype,
                                                       device=X_local.device)
        ops = []
        for r in range(world):
            if r == dst or counts[r] == 0:
                continue
            ops.append(dist.P2POp(dist.irecv, Xall[offs[r]:offs[r + 1]], dist.get_global_rank(
                group, r) if group is not None else r, group=group))
        if counts[dst]:
            Xall[offs[dst]:offs[dst + 1]].copy_(X_local[: counts[dst]])
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        return Xall
    if counts[rank]:  # the same batched P2P API on both sides (one NCCL group per call)
        peer = dist.get_global_rank(group, dst) if group is not None else dst
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, X_local[: counts[rank]].contiguous(),
                                                    peer, group=group)]):
            w.wait()
    return None


def hsrq3in_distributed(h, eigenvalues, config=None, group=None, device=None, dst=0,
                        solve_fn=None):
    """hsrq3in (inviter.py:186-254) with the selection sharded over the ranks.

    Each rank runs the restart loop (inviter._iterate_mixed) on its shard with
    its own sweep; the ranks iterate in lockstep and raise the reference's
    first failure everywhere.  Returns the full EigvecResult (caller order,
    scale exponents and log2 norms included) on ``dst``, None elsewhere.
    ``solve_fn`` replaces solver.solve_group (tests run the driver on CPU
    ranks with the oracle standing in for the GPU).
    """
    from .core import ConfigError
    from .inviter import EigvecResult, InviterConfig, _iterate_mixed, device_hessenberg

    config = config or InviterConfig()
    if config.w_max is not None:
        raise ConfigError("hsrq3in_distributed does not take a w_max cap (each rank solves its "
                          "shard in one group)")
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    eigs = np.asarray(eigenvalues, dtype=np.complex128).ravel()
    if eigs.size == 0:
        raise ConfigError("empty eigenvalue selection")
    m = eigs.size
    is_cplx = eigs.imag != 0.0
    m1 = int(np.count_nonzero(~is_cplx))
    # position of every shift in its reference call (real-first stable order)
    call_pos = np.empty(m, dtype=np.int64)
    call_pos[~is_cplx] = np.arange(m1)
    call_pos[is_cplx] = np.arange(m - m1)
    idx, mine = local_selection(eigs, rank, world)
    mine_r = ~(mine.imag != 0.0)
    ir, ic = idx[mine_r], idx[~mine_r]
    ec = eigs[ic]
    flip = ec.imag < 0.0
    canon = np.where(flip, ec.conj(), ec)
    ex = ShardExchange(group, call_pos[ir], call_pos[ic])
    try:
        dh = device_hessenberg(h, device)
        s = _iterate_mixed(dh, eigs[ir].real, canon, config, device, exchange=ex, solve_fn=solve_fn)
    except (HessrqError, ShardError):
        raise  # raised alike on every rank (same inputs / the exchange)
    except Exception as e:  # noqa: BLE001 - announce, then fail everywhere
        ex.poison(e)
        raise
    ncol = 0 if s.X is None else int(s.X.shape[0])
    R, C = s.meta["real"], s.meta["cplx"]
    payload = dict(ncol=ncol, ir=ir, ic=ic, col_r=s.col_r, col_c=s.col_c, flip=flip,
                   meta={k: (R[k], C[k]) for k in ("conv", "restarts", "norms", "log2", "aexp", "seg")},
                   launches=s.launches)
    allp = ex.collect(payload)
    counts = [p["ncol"] for p in allp]
    n = dh.n
    Xl = s.X if s.X is not None else torch.empty((0, n), dtype=torch.float64,
                                                 device=dh.t.device if hasattr(dh, "t") else "cpu")
    Xall = gather_columns(Xl, counts, group=group, dst=dst)
    if rank != dst:
        return None
    N = s.N
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    re_col = np.empty(m, np.int64)
    im_col = np.full(m, -1, np.int64)
    sgn = np.ones(m)
    conv = np.zeros(m, dtype=bool)
    restarts = np.zeros(m, dtype=np.int64)
    norms = np.zeros(m)
    log2n = np.full(m, -np.inf)
    aexp = np.zeros(m, dtype=np.int32)
    seg = np.zeros((N, m), dtype=np.int32)
    launches = 0
    for r, p in enumerate(allp):
        launches += p["launches"]
        for kind, gidx, cols in ((0, p["ir"], p["col_r"]), (1, p["ic"], p["col_c"])):
            if gidx.size == 0:
                continue
            re_col[gidx] = offs[r] + cols
            if kind == 1:
                im_col[gidx] = offs[r] + cols + 1
                sgn[gidx] = np.where(p["flip"], -1.0, 1.0)
            M = p["meta"]
            conv[gidx] = M["conv"][kind]
            restarts[gidx] = M["restarts"][kind]
            norms[gidx] = M["norms"][kind]
            log2n[gidx] = M["log2"][kind]
            aexp[gidx] = M["aexp"][kind]
            seg[:, gidx] = M["seg"][kind]
    vectors = _assemble(Xall, re_col, im_col, sgn, n)
    res = EigvecResult(vectors=vectors, converged=conv, restarts=restarts, norms=norms,
                       eigenvalues=eigs.copy(), alpha=np.ldexp(1.0, aexp), alpha_exp=aexp,
                       segment_scales=np.ldexp(1.0, seg), segment_exp=seg, log2_norms=log2n,
                       extras={"gpu_launches": launches, "ranks": world,
                               "gathered_bytes": int(8 * n * (offs[-1] - counts[dst]))})
    res.peak_crossover_reals = max(n * N * m1, 2 * n * N * (m - m1))
    return res


def _assemble(Xall, re_col, im_col, sgn, n):
    """Caller-order (n, m) complex128 vectors from the gathered block: on the
    GPU through hsrq_pack_download; a CPU block (gloo tests) with torch ops."""
    if Xall.is_cuda:
        from .inviter import _pack, _Solved

        s = _Solved(dh=_NStub(n), X=Xall, col_r=None, col_c=None, meta=None, launches=0, N=0)
        return _pack(s, re_col, im_col, sgn, True)
    re = Xall[torch.from_numpy(re_col)].numpy()
    im = np.zeros_like(re)
    has = im_col >= 0
    im[has] = Xall[torch.from_numpy(im_col[has])].numpy() * sgn[has][:, None]
    return np.ascontiguousarray((re + 1j * im).T)


class _NStub:
    def __init__(self, n):
        self.n = n
