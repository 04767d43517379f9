"""World-size-2 runs of the sharded driver (parallel.hsrq3in_distributed) over
gloo on CPU ranks.

The per-attempt solve is injected (``solve_fn``): the CPU oracle stands in for
each rank's GPU sweep (test-only), and the matrix for the device copy of H.
Everything else is the production path: the shard selection, the lockstep
restart loop of inviter._iterate_mixed with its per-attempt exchange, the
failure exchange that makes every rank raise the reference's first failure,
the poison path (an exception on one rank must not leave the other waiting in
a collective), and the point-to-point gather of the solution columns to rank
0 (real columns once, complex shifts as re/im pairs: exactly X's bytes).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

N_MAT = 40
B_R = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance():
    rng = np.random.default_rng(0)
    n = N_MAT
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    ev = np.linalg.eigvals(h)
    sel = np.concatenate([ev[ev.imag > 0][:3], ev[ev.imag == 0][:4], ev[ev.imag < 0][:2],
                          ev[ev.imag == 0][4:6], ev[ev.imag > 0][3:5]])
    return h, sel


class StandInH:
    """The device copy of H, for CPU ranks (infinity norm / unreducedness as
    HessenbergMatrix computes them)."""

    is_device_stand_in = True

    def __init__(self, h):
        from paper_2101_05063_b200.core import HessenbergMatrix

        hm = HessenbergMatrix(h)
        self.h, self.n = hm.data, hm.n
        self._norm, self._unred = hm.infinity_norm(), hm.is_unreduced()

    def infinity_norm(self):
        return self._norm

    def is_unreduced(self):
        return self._unred


class _Out:
    pass


class _GS:
    pass


def make_solve_fn(bad=(), singular=(), crash=None):
    """solve_group stand-in on the oracle.  ``bad``: shifts whose first attempt
    is reported unconverged (forces a restart); ``singular``: shifts reported
    as an exactly singular factor (packed code, tile 2, row 3); ``crash``: a
    shift whose solve raises (a device failure on that rank)."""
    bad = [complex(z) for z in bad]
    singular = [complex(z) for z in singular]

    def solve_fn(dh, ec, er, start, b_r, **kw):
        import sys

        sys.path.insert(0, ROOT)
        from oracle import oracle as O

        h, n = dh.h, dh.n
        ec = np.asarray(ec, dtype=np.complex128)
        er = np.asarray(er, dtype=np.float64)
        lams = np.concatenate([ec, er.astype(complex)])
        if crash is not None and np.any(lams == crash):
            raise RuntimeError("simulated device failure")
        first = bool(np.all(start == start[0]))
        parts = []
        if ec.size:
            parts.append(O.solve(h, ec, np.repeat(start[:, None], ec.size, 1).astype(complex), b_r,
                                 mode="eigvec"))
        if er.size:
            parts.append(O.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, mode="eigvec"))
        X = np.zeros((2 * ec.size + er.size, n))
        if ec.size:
            X[0:2 * ec.size:2] = parts[0].x.real.T
            X[1:2 * ec.size:2] = parts[0].x.imag.T
        if er.size:
            X[2 * ec.size:] = parts[-1].x.T
        out = _Out()
        cat = lambda f: np.concatenate([getattr(p, f) for p in parts], axis=-1)
        norms = cat("norms").copy()
        fail = np.zeros(lams.size, dtype=np.int64)
        for q, z in enumerate(lams):
            if first and z in bad:
                norms[q] = 0.0
            if z in singular:
                fail[q] = (2 << 56) | (2 << 24) | 3
        out.X = torch.from_numpy(X)
        out.fail = torch.from_numpy(fail)
        out.nfail = int(np.count_nonzero(fail))
        out.norms = torch.from_numpy(norms)
        out.log2norm = torch.from_numpy(cat("log2norm"))
        out.alpha_exp = torch.from_numpy(cat("alpha_exp"))
        out.seg_exp = torch.from_numpy(cat("segment_exp"))
        out.launches = 0
        out.perm = None
        gs = _GS()
        gs.X = out.X
        return out, gs

    return solve_fn


def _expected(h, sel, bad):
    """Per caller column: the oracle's vector for the start vector of the
    attempt that converged (attempt 1 for the forced restarts)."""
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2101_05063_b200.inviter import InviterConfig, _next_start

    n = h.shape[0]
    rho = np.finfo(float).eps * StandInH(h).infinity_norm()
    s0 = rho * np.ones(n)
    s1 = _next_start(rho, n, [s0.copy()], InviterConfig().restart_seed, 1)
    want = np.zeros((n, sel.size), dtype=complex)
    for j, z in enumerate(sel):
        st = s1 if complex(z) in [complex(b) for b in bad] or complex(np.conj(z)) in \
            [complex(b) for b in bad] else s0
        if z.imag == 0:
            want[:, j] = O.solve(h, np.array([z.real]), st[:, None], B_R, mode="eigvec").x[:, 0]
        else:
            c = z if z.imag > 0 else np.conj(z)
            x = O.solve(h, np.array([c]), st[:, None].astype(complex), B_R, mode="eigvec").x[:, 0]
            want[:, j] = x if z.imag > 0 else np.conj(x)
    return want


def _worker(rank, world, port, out, case):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2101_05063_b200 import InviterConfig, SingularSystemError
    from paper_2101_05063_b200.parallel import ShardError, hsrq3in_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, sel = _instance()
    cfg = InviterConfig(b_r=B_R, b_c=2)
    res = {}
    try:
        if case == "restart":
            bad = [sel[1], sel[4]]  # one complex, one real shift restart once
            r = hsrq3in_distributed(StandInH(h), sel, cfg, solve_fn=make_solve_fn(bad=bad))
            if rank == 0:
                want = _expected(h, sel, bad)
                res = dict(err=float(np.abs(r.vectors - want).max()), conv=bool(r.converged.all()),
                           restarts=r.restarts.tolist(), bytes=r.extras["gathered_bytes"])
            else:
                res = dict(none=r is None)
        elif case == "singular":
            try:
                hsrq3in_distributed(StandInH(h), sel, cfg,
                                    solve_fn=make_solve_fn(singular=[sel[5], np.conj(sel[7])]))
                res = dict(raised=None)
            except SingularSystemError as e:
                res = dict(raised=(e.shift_index, e.local_index))
        elif case == "crash":
            try:
                hsrq3in_distributed(StandInH(h), sel, cfg,
                                    solve_fn=make_solve_fn(crash=sel[2]))
                res = dict(raised=None)
            except ShardError as e:
                res = dict(raised="shard", msg=str(e))
    finally:
        np.save(out + f".{rank}.npy", np.array([res], dtype=object), allow_pickle=True)
        dist.destroy_process_group()


def _run(tmp_path, case):
    out = str(tmp_path / case)
    ctx = mp.spawn(_worker, args=(2, _free_port(), out, case), nprocs=2, join=False)
    assert ctx.join(timeout=240) or ctx.join(timeout=60), "ranks did not finish (hang)"
    return [np.load(out + f".{r}.npy", allow_pickle=True)[0] for r in range(2)]


def test_sharded_restarts_and_gather_match_single_process(tmp_path):
    r0, r1 = _run(tmp_path, "restart")
    assert r1["none"]
    assert r0["err"] <= 1e-13 and r0["conv"]
    h, sel = _instance()
    canon = np.where(sel.imag < 0, sel.conj(), sel)
    want_r = [1 if canon[j] in (sel[1], sel[4]) else 0 for j in range(sel.size)]
    assert sum(want_r) == 3  # sel[8] is sel[1]'s conjugate: the same solve
    assert r0["restarts"] == want_r
    # rank 1's block crossed once: its real columns + complex pairs
    n = N_MAT
    is_c = sel.imag != 0
    from paper_2101_05063_b200.parallel import local_selection

    idx, mine = local_selection(sel, 1, 2)
    cols = int(np.count_nonzero(mine.imag == 0) + 2 * np.count_nonzero(mine.imag != 0))
    assert r0["bytes"] == 8 * n * cols and is_c.any()


def test_sharded_failure_raises_reference_first_failure_everywhere(tmp_path):
    """Both ranks raise the SingularSystemError the single-process driver
    raises (the reference's order: the real call before the complex one)."""
    import sys

    sys.path.insert(0, ROOT)
    from paper_2101_05063_b200 import InviterConfig, SingularSystemError
    from paper_2101_05063_b200.inviter import _iterate_mixed

    r0, r1 = _run(tmp_path, "singular")
    h, sel = _instance()
    is_c = sel.imag != 0
    er = sel[~is_c].real
    ec = sel[is_c]
    ec = np.where(ec.imag < 0, ec.conj(), ec)
    with pytest.raises(SingularSystemError) as e:
        _iterate_mixed(StandInH(h), er, ec, InviterConfig(b_r=B_R, b_c=2),
                       solve_fn=make_solve_fn(singular=[sel[5], np.conj(sel[7])]))
    assert r0["raised"] == r1["raised"] == (e.value.shift_index, e.value.local_index)


def test_sharded_crash_on_one_rank_fails_every_rank(tmp_path):
    r0, r1 = _run(tmp_path, "crash")
    assert r0["raised"] == r1["raised"] == "shard"
    assert "simulated device failure" in r0["msg"]
