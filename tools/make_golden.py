"""Generate tests/golden/*.npz from the LIVE reference (hessrq, numba backend).

Run in the build container, where /root/reference exists:
    python tools/make_golden.py
The fixtures pin the CPU oracle (oracle/) and the GPU path to the reference's
own outputs: tile kernels, scalar helpers, full dhsrq3/chsrq3 solves (robust,
non-robust, solve/eigvec modes, ragged tiles, the H2 overflow fixture of
verifysuite.py:107-124), the inverse-iteration drivers and BASELINE config 1.
"""

from __future__ import annotations

import ctypes
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import hessrq  # noqa: E402
from hessrq import _kernels  # noqa: E402
from hessrq.backsolve import chsrq3, dhsrq3  # noqa: E402
from hessrq.inviter import InviterConfig, _next_start, chsrq3in, dhsrq3in, hsrq3in  # noqa: E402
from hessrq.testprob import gen_h1, gen_h2, gen_h3, uniform_open_closed  # noqa: E402
from hessrq.verifysuite import random_unreduced  # noqa: E402

assert hessrq.backend_name() == "numba", "numba backend required (see SURVEY.md §0 finding 5)"
K = _kernels.get_backend()
_DMAX = float(np.finfo(np.float64).max)


def blas_corename():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    return O.blas_corename()


def save(name, **arrs):
    os.makedirs(OUT, exist_ok=True)
    arrs["corename"] = np.array(blas_corename())
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)


def gen_scalars():
    rng = np.random.default_rng(7)
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    e1 = rng.integers(-1070, 1020, 4000)
    e2 = np.clip(e1 + rng.integers(-60, 60, 4000), -1074, 1023)
    hx = rng.uniform(-1, 1, 4000) * np.ldexp(1.0, e1)
    hy = rng.uniform(-1, 1, 4000) * np.ldexp(1.0, e2)
    hx[:8] = [0.0, 3.0, 1e308, 5e-324, -0.0, 1.0, 2.0 ** 511, 2.0 ** -511]
    hy[:8] = [0.0, 4.0, 1e308, 5e-324, 7.0, 1e-20, 3.0, 2.0 ** -600]
    hyp = np.array([libm.hypot(a, b) for a, b in zip(hx, hy)])
    omega = _DMAX / 2.0 / 128
    pb = np.abs(rng.standard_normal(3000)) * np.ldexp(1.0, rng.integers(-20, 1024, 3000))
    ph = np.abs(rng.standard_normal(3000)) * np.ldexp(1.0, rng.integers(-20, 600, 3000))
    px = np.abs(rng.standard_normal(3000)) * np.ldexp(1.0, rng.integers(-300, 700, 3000))
    pb = np.where(np.isfinite(pb), pb, 1e300)
    pu = np.array([K.protect_update(a, b, c, omega) for a, b, c in zip(pb, ph, px)])
    f2 = np.abs(rng.standard_normal(500)) * np.ldexp(1.0, rng.integers(-1074, 1000, 500))
    f2[:4] = [0.0, -1.0, np.inf, 5e-324]
    p2f = np.array([K.pow2floor(v) for v in f2])
    seeds = np.array([0x5EED, 0x5EED + 0x9E37, 12345, 2**63 + 17], dtype=np.uint64)
    uoc = np.stack([uniform_open_closed(int(s), 64) for s in seeds])
    # restart vectors, inviter.py:76-88
    n = 37
    rho = 1e-14
    prev = [rho * np.ones(n)]
    starts = []
    for att in (1, 2, 3):
        v = _next_start(rho, n, prev, 0x5EED, att)
        prev.append(v.copy())
        starts.append(v)
    save("scalars", hx=hx, hy=hy, hypot=hyp, pb=pb, ph=ph, px=px, omega=np.float64(omega),
         protect=pu, p2in=f2, p2out=p2f, seeds=seeds, uoc=uoc, starts=np.stack(starts))


def gen_tiles():
    rng = np.random.default_rng(11)
    cases = {}
    idx = 0
    for k, b, has_left, small_omega in ((16, 3, True, False), (37, 4, False, False),
                                        (128, 3, True, False), (64, 5, True, True),
                                        (128, 2, False, True), (1, 2, True, False),
                                        (2, 3, False, False)):
        h = random_unreduced(max(k, 2) + 1, 100 + idx).data
        hdiag = np.ascontiguousarray(h[1 : k + 1, 1:k])
        hleft = np.ascontiguousarray(h[1 : k + 1, 0])
        lam = rng.uniform(-3, 3, b)
        rright = rng.standard_normal((k, b))
        xin = rng.standard_normal((k, b)) * (1e300 if small_omega else 1.0)
        omega = 1e10 if small_omega else _DMAX / 2.0 / 128
        c = np.empty((k, b))
        s = np.empty((k, b))
        st_r = K.reduce_diag(hdiag, hleft, has_left, lam, rright, c, s)
        x = xin.copy()
        beta = np.ones(b)
        st_s = K.solve_rsolve(hdiag, hleft, has_left, lam, rright, c, s, x, beta, True, omega)
        # complex
        clr, cli = rng.uniform(-3, 3, b), rng.uniform(0.1, 3, b)
        rr2 = rng.standard_normal((k, 2 * b))
        x2in = rng.standard_normal((k, 2 * b)) * (1e300 if small_omega else 1.0)
        cre, cim, cs = np.empty((k, b)), np.empty((k, b)), np.empty((k, b))
        st_cr = K.creduce_diag(hdiag, hleft, has_left, clr, cli, rr2, cre, cim, cs)
        x2 = x2in.copy()
        cbeta = np.ones(b)
        st_cs = K.csolve_crsolve(hdiag, hleft, has_left, clr, cli, rr2, cre, cim, cs, x2, cbeta,
                                 True, omega)
        cases.update({
            f"t{idx}_meta": np.array([k, b, int(has_left), int(st_r), int(st_s), int(st_cr),
                                      int(st_cs)], dtype=np.int64),
            f"t{idx}_omega": np.float64(omega),
            f"t{idx}_hdiag": hdiag, f"t{idx}_hleft": hleft, f"t{idx}_lam": lam,
            f"t{idx}_rright": rright, f"t{idx}_xin": xin, f"t{idx}_c": c, f"t{idx}_s": s,
            f"t{idx}_x": x, f"t{idx}_beta": beta, f"t{idx}_clr": clr, f"t{idx}_cli": cli,
            f"t{idx}_rr2": rr2, f"t{idx}_x2in": x2in, f"t{idx}_cre": cre, f"t{idx}_cim": cim,
            f"t{idx}_cs": cs, f"t{idx}_x2": x2, f"t{idx}_cbeta": cbeta,
        })
        idx += 1
    save("tiles", ntiles=np.int64(idx), **cases)


def _solve_case(store, tag, h, lam, b, b_r, b_c, robust, mode, cplx):
    f = chsrq3 if cplx else dhsrq3
    r = f(h, lam, b, b_r=b_r, b_c=b_c, robust=robust, mode=mode)
    store[f"{tag}_h"] = np.asfortranarray(h.data if hasattr(h, "data") else h)
    store[f"{tag}_lam"] = lam
    store[f"{tag}_b"] = b
    store[f"{tag}_cfg"] = np.array([b_r, b_c, int(robust), {"solve": 0, "eigvec": 1}[mode],
                                    int(cplx)], dtype=np.int64)
    store[f"{tag}_x"] = r.x
    store[f"{tag}_alpha"] = r.alpha
    store[f"{tag}_seg"] = r.segment_scales.alpha
    store[f"{tag}_norms"] = r.norms if r.norms is not None else np.full(len(lam), np.nan)


def gen_solves():
    store = {}
    tags = []
    rng = np.random.default_rng(3)
    specs = [(24, 6, 2, 1), (70, 16, 5, 2), (64, 64, 3, 3), (33, 8, 32, 4), (129, 32, 7, 5),
             (200, 128, 16, 6), (40, 5, 1, 7)]
    for n, b_r, b_c, seed in specs:
        h = random_unreduced(n, seed)
        nrm = h.infinity_norm()
        lam = nrm * rng.uniform(-2, 2, 6)
        b = rng.standard_normal((n, 6))
        clam = nrm * (rng.uniform(-2, 2, 4) + 1j * rng.uniform(0.05, 2, 4))
        cb = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
        for robust, mode in ((True, "solve"), (True, "eigvec"), (False, "solve")):
            t = f"s{len(tags)}"
            _solve_case(store, t, h, lam, b, b_r, b_c, robust, mode, False)
            tags.append(t)
            t = f"s{len(tags)}"
            _solve_case(store, t, h, clam, cb, b_r, b_c, robust, mode, True)
            tags.append(t)
    # overflow fixture (verifysuite.py:107-124)
    for b_r in (16, 7, 60):
        t = f"s{len(tags)}"
        _solve_case(store, t, gen_h2(60), np.array([2.0]), 1e290 * np.ones((60, 1)), b_r, 1, True,
                    "solve", False)
        tags.append(t)
    t = f"s{len(tags)}"
    _solve_case(store, t, gen_h2(60), np.array([2.0 + 0.5j]), 1e290 * np.ones((60, 1)) + 0j, 16,
                1, True, "solve", True)
    tags.append(t)
    t = f"s{len(tags)}"
    _solve_case(store, t, gen_h3(60), np.array([2.0]), np.ones((60, 1)), 16, 1, True, "solve",
                False)
    tags.append(t)
    save("solves", tags=np.array(tags), **store)


def gen_budget():
    """dhsrq3 / chsrq3 with a caller's OverflowBudget (backsolve.py:342-346):
    small omegas make every guard fire at ordinary magnitudes."""
    from hessrq.overflow import OverflowBudget

    store = {}
    tags = []
    rng = np.random.default_rng(11)
    for n, b_r, seed in ((48, 16, 1), (70, 32, 2), (65, 64, 3)):
        h = random_unreduced(n, seed)
        nrm = h.infinity_norm()
        lam = nrm * rng.uniform(-1, 1, 3)  # well-conditioned systems: the guards fire
        clam = nrm * (rng.uniform(-1, 1, 3) + 1j * rng.uniform(0.05, 1, 3))  # because omega is small
        b = rng.standard_normal((n, lam.size))
        cb = rng.standard_normal((n, clam.size)) + 1j * rng.standard_normal((n, clam.size))
        for omega in (1.0, 8.0, 1e3, 2.0 ** 600):
            for mode in ("solve", "eigvec"):
                for cplx, L, B in ((False, lam, b), (True, clam, cb)):
                    if L.size == 0:
                        continue
                    f = chsrq3 if cplx else dhsrq3
                    r = f(h, L, B, b_r=b_r, b_c=2, robust=True, mode=mode,
                          budget=OverflowBudget(omega=omega))
                    t = f"b{len(tags)}"
                    store[f"{t}_h"] = np.asfortranarray(h.data)
                    store[f"{t}_lam"] = L
                    store[f"{t}_b"] = B
                    store[f"{t}_cfg"] = np.array([b_r, 2, {"solve": 0, "eigvec": 1}[mode],
                                                  int(cplx)], dtype=np.int64)
                    store[f"{t}_omega"] = np.array(omega)
                    store[f"{t}_x"] = r.x
                    store[f"{t}_alpha"] = r.alpha
                    store[f"{t}_seg"] = r.segment_scales.alpha
                    store[f"{t}_norms"] = r.norms if r.norms is not None else np.full(L.size, np.nan)
                    tags.append(t)
    save("budget", tags=np.array(tags), **store)


def gen_update_tiles():
    """update_rupdate / cupdate_crupdate and reduce_offdiag / creduce_offdiag
    on single tiles (numba_backend.py:109-125, 198-311, 467-490, 579-736):
    tile shapes of full, short (ragged last tile) and odd heights, shifted
    and far tiles, robust and plain, magnitudes where every guard fires."""
    store = {}
    tags = []
    rng = np.random.default_rng(21)
    for m, k in ((128, 128), (128, 77), (64, 64), (37, 21)):
        for cplx in (False, True):
            for shifted in (True, False):
                for robust, scale in ((True, 1.0), (True, 1e300), (False, 1.0)):
                    b = 5
                    ht = rng.standard_normal((m, k))
                    th = rng.uniform(0, 2 * np.pi, (k, b))
                    if cplx:
                        ph = rng.uniform(0, 2 * np.pi, (k, b))
                        cre, cim, s = np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), np.sin(th)
                        lre, lim = rng.standard_normal(b), rng.uniform(0.1, 2, b)
                        rr = rng.standard_normal((m, 2 * b))
                        xb = scale * rng.standard_normal((k, 2 * b))
                        bio = scale * rng.standard_normal((m, 2 * b))
                    else:
                        cre, cim, s = np.cos(th), None, np.sin(th)
                        lre, lim = rng.standard_normal(b), None
                        rr = rng.standard_normal((m, b))
                        xb = scale * rng.standard_normal((k, b))
                        bio = scale * rng.standard_normal((m, b))
                    aexp = rng.integers(-6, 1, b).astype(np.int32)
                    bexp = rng.integers(-6, 1, b).astype(np.int32)
                    alpha, beta = np.ldexp(1.0, aexp), np.ldexp(1.0, bexp)
                    omega = _DMAX / 2.0 / m if robust else math.inf
                    lz = lre if shifted else np.zeros(b)
                    lzi = (lim if shifted else np.zeros(b)) if cplx else None
                    bo = bio.copy()
                    bt = beta.copy()
                    rl = np.empty_like(rr)
                    if cplx:
                        K.cupdate_crupdate(ht, rr, alpha, xb, lz, lzi, shifted, cre, cim, s, bt, bo,
                                           robust, omega)
                        K.creduce_offdiag(ht, lz, lzi, cre, cim, s, rr, rl)
                    else:
                        K.update_rupdate(ht, rr, alpha, xb, lz, shifted, cre, s, bt, bo, robust,
                                         omega)
                        K.reduce_offdiag(ht, lz, cre, s, rr, rl)
                    t = f"u{len(tags)}"
                    store.update({f"{t}_cfg": np.array([m, k, b, int(cplx), int(shifted),
                                                        int(robust)], dtype=np.int64),
                                  f"{t}_ht": ht, f"{t}_rr": rr, f"{t}_aexp": aexp, f"{t}_xb": xb,
                                  f"{t}_lre": lre, f"{t}_cre": cre, f"{t}_s": s, f"{t}_bexp": bexp,
                                  f"{t}_bio": bio, f"{t}_out_b": bo, f"{t}_out_beta": bt,
                                  f"{t}_out_rleft": rl})
                    if cplx:
                        store.update({f"{t}_lim": lim, f"{t}_cim": cim})
                    tags.append(t)
    save("update_tiles", tags=np.array(tags), **store)


def gen_inviter():
    store = {}
    # H1 with known eigenvalues, real and complex parts
    h, eigs = gen_h1(32, 0.5, seed=4)
    cfg = InviterConfig(b_r=8, b_c=4)
    r = hsrq3in(h, eigs, cfg)
    store.update(h1_h=np.asfortranarray(h.data), h1_eigs=eigs, h1_vectors=r.vectors,
                 h1_conv=r.converged, h1_restarts=r.restarts, h1_norms=r.norms)
    sel = eigs[eigs.imag > 0]
    rc = chsrq3in(h, sel.conj(), cfg)
    store.update(h1c_vectors=rc.vectors, h1c_norms=rc.norms)
    rr = dhsrq3in(h, eigs[eigs.imag == 0].real, cfg)
    store.update(h1r_vectors=rr.vectors, h1r_norms=rr.norms, h1r_restarts=rr.restarts)
    # a case with restarts: shifts exactly at eigenvalues of a tiny matrix + far shift
    h2 = random_unreduced(20, 5)
    ev = np.linalg.eigvals(h2.data)
    shifts = np.concatenate([ev[np.abs(ev.imag) == 0].real[:3], [1e3]])
    r2 = dhsrq3in(h2, shifts, InviterConfig(b_r=5, b_c=2))
    store.update(rs_h=np.asfortranarray(h2.data), rs_shifts=shifts, rs_vectors=r2.vectors,
                 rs_conv=r2.converged, rs_restarts=r2.restarts, rs_norms=r2.norms)
    # BASELINE config 1 (n=256, all real, b_r=32): dhsrq3in through hsrq3in
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import instances

    h1 = instances.make_h(1)
    s1 = instances.shifts(1)
    r1 = hsrq3in(h1, s1, InviterConfig(b_r=32))
    store.update(c1_h=h1, c1_shifts=s1, c1_vectors=r1.vectors.real, c1_conv=r1.converged,
                 c1_restarts=r1.restarts, c1_norms=r1.norms)
    save("inviter", **store)


_NODE_KINDS = ["ReduceDiag", "SolveTile", "MergedSolveBacktransform"]


def _reference_error(f):
    """The SingularSystemError a reference call raises (unwrapping TaskError), or None.
    The error carries ``task`` = (kind index in _NODE_KINDS, tile_i, tile_j, batch,
    seq) of the TaskError's node (scheduler.py:182-187) and ``task_message``."""
    from hessrq.core import SingularSystemError
    from hessrq.scheduler import TaskError

    try:
        f()
    except Exception as e:  # noqa: BLE001 - scheduler wraps the kernel error in TaskError
        c = e
        while c is not None and not isinstance(c, SingularSystemError):
            c = c.__cause__
        if c is None:
            raise
        assert isinstance(e, TaskError) and e.cause is c and e.__cause__ is c
        c.task = (_NODE_KINDS.index(e.node.kind),) + tuple(e.node.coords) + (e.node.seq,)
        c.task_message = str(e)
        return c
    return None


def gen_singular():
    """Exactly singular shifted systems (SingularSystemError parity).

    Small-integer Hessenberg matrices with an integer (real case) or Gaussian
    integer (complex case) eigenvalue: the shifted matrix is exactly singular
    and the reference's final pivot is exactly 0.0.  Recorded per case: the
    shift_index / local_index the reference reports (backsolve.py:53-59),
    for the solver and for the inverse-iteration driver.
    """
    store = {}
    tags = []
    rng = np.random.default_rng(3)
    n = 8
    want_real, want_cplx = 4, 2
    for trial in range(20000):
        if want_real == 0 and want_cplx == 0:
            break
        h = np.triu(rng.integers(-2, 3, (n, n))).astype(float)
        h[np.arange(1, n), np.arange(n - 1)] = rng.choice([-2.0, -1.0, 1.0, 2.0], n - 1)
        ev = np.linalg.eigvals(h)
        for lam in ev:
            lr, li = round(lam.real), round(lam.imag)
            if abs(lam - complex(lr, li)) > 1e-9:
                continue
            cplx = li != 0
            if (cplx and (want_cplx == 0 or li < 0)) or (not cplx and want_real == 0):
                continue
            z = complex(lr, li)
            lam_v = (np.array([z + 0.25, z, z + 0.5j if cplx else z + 0.5, z]) if cplx
                     else np.array([lr + 0.25, lr, lr + 0.5, lr], dtype=float))
            b = np.ones((n, 4)) + (0j if cplx else 0)
            f = chsrq3 if cplx else dhsrq3
            hit, nodes, msgs = [], [], []
            for b_r, b_c in ((8, 4), (3, 2), (2, 1)):
                e = _reference_error(lambda: f(h, lam_v, b, b_r=b_r, b_c=b_c))
                if e is not None:
                    hit.append((b_r, b_c, e.shift_index, e.local_index))
                    nodes.append(e.task)
                    msgs.append(e.task_message)
            if not hit:
                continue
            ei = _reference_error(lambda: hsrq3in(h, np.array([z]), InviterConfig(b_r=3, b_c=2)))
            t = f"g{len(tags)}"
            store[f"{t}_h"] = np.asfortranarray(h)
            store[f"{t}_lam"] = lam_v
            store[f"{t}_cplx"] = np.array(int(cplx))
            store[f"{t}_hits"] = np.array(hit, dtype=np.int64)
            store[f"{t}_inviter"] = np.array(
                [-1, -1] if ei is None else [ei.shift_index, ei.local_index], dtype=np.int64)
            # the TaskError the caller actually sees (scheduler.py:182-187, 211-214):
            # node (kind index, tile_i, tile_j, batch, seq) and its message, per hit
            store[f"{t}_nodes"] = np.array(nodes, dtype=np.int64)
            store[f"{t}_messages"] = np.array(msgs)
            store[f"{t}_inviter_node"] = np.array(
                [-1] * 5 if ei is None else list(ei.task), dtype=np.int64)
            store[f"{t}_inviter_message"] = np.array("" if ei is None else ei.task_message)
            tags.append(t)
            if cplx:
                want_cplx -= 1
            else:
                want_real -= 1
            break
    # seq of the nodes a failure can surface in, from the reference's own graph
    # builders (scheduler.py:120-179): [N - 1, batch, tile] for N = 1..5, 3 batches
    from types import SimpleNamespace

    from hessrq.scheduler import build_reduce_dag, build_solve_dag

    rseq = -np.ones((5, 3, 5), dtype=np.int64)
    sseq = -np.ones((5, 3, 5), dtype=np.int64)
    for N in range(1, 6):
        gr = build_reduce_dag(SimpleNamespace(N=N), 3)
        gs = build_solve_dag(SimpleNamespace(N=N), 3)
        for node in gr.nodes:
            if node.kind == "ReduceDiag":
                rseq[N - 1, node.coords[2], node.coords[0]] = node.seq
        for node in gs.nodes:
            if node.kind in ("SolveTile", "MergedSolveBacktransform"):
                sseq[N - 1, node.coords[2], node.coords[0]] = node.seq
    save("singular", tags=np.array(tags), node_kinds=np.array(_NODE_KINDS), dag_reduce_seq=rseq,
         dag_solve_seq=sseq, **store)


def gen_edge():
    """Edge inputs of the inverse-iteration drivers (inviter.py:109-254): n = 1,
    2, 3, a one-row ragged last tile (n = 33, b_r = 32), one shift of either
    kind, only Im < 0 shifts, a repeated shift, the caller's mixed order, an
    empty selection -- what the reference returns or raises for each."""
    rng = np.random.default_rng(11)
    store, tags = {}, []

    def case(tag, h, eigs, b_r, fn=hsrq3in):
        store[f"{tag}_h"] = np.asfortranarray(h)
        store[f"{tag}_eigs"] = np.asarray(eigs)
        store[f"{tag}_br"] = np.array(b_r)
        store[f"{tag}_fn"] = np.array(fn.__name__)
        try:
            r = fn(h, eigs, InviterConfig(b_r=b_r))
        except Exception as e:  # noqa: BLE001 - the reference's error is the fixture
            store[f"{tag}_error"] = np.array(type(e).__name__)
            store[f"{tag}_message"] = np.array(str(e))
        else:
            store[f"{tag}_error"] = np.array("")
            v = np.asarray(r.vectors)
            store[f"{tag}_vectors"] = v.astype(np.complex128)
            store[f"{tag}_conv"] = np.asarray(r.converged)
            store[f"{tag}_restarts"] = np.asarray(r.restarts)
        tags.append(tag)

    def hess(n):
        h = np.triu(rng.standard_normal((n, n)), -1)
        for i in range(1, n):
            h[i, i - 1] = abs(h[i, i - 1]) + 0.1
        return h

    case("n1_exact", np.array([[2.0]]), np.array([2.0]), 1)
    case("n1_near", np.array([[2.0]]), np.array([2.0 + 1e-9]), 1)
    h2 = hess(2)
    case("n2_all", h2, np.linalg.eigvals(h2), 2)
    h3 = hess(3)
    case("n3_all", h3, np.linalg.eigvals(h3), 2)  # ragged: tiles of 2 + 1
    h33 = hess(33)
    ev = np.linalg.eigvals(h33)
    er, ec = ev[ev.imag == 0], ev[ev.imag > 0]
    case("n33_ragged", h33, ev, 32)
    case("n33_one_real", h33, er[:1].real, 32, dhsrq3in)
    case("n33_one_cplx", h33, ec[:1], 32, chsrq3in)
    case("n33_conj_only", h33, np.conj(ec[:3]), 32)
    case("n33_repeated", h33, np.array([ec[0], er[0], ec[0], er[0]]), 32)
    case("n33_mixed_order", h33, np.concatenate([np.conj(ec[:2]), er[:2], ec[:2]])[::-1], 32)
    case("n33_empty", h33, ev[:0], 32)
    case("n33_empty_real", h33, er[:0].real, 32, dhsrq3in)
    case("n33_real_as_complex_api", h33, er[:2].astype(complex), 32, chsrq3in)
    case("n33_complex_to_real_api", h33, ec[:1], 32, dhsrq3in)
    save("edge", tags=np.array(tags), **store)


def gen_backtransform():
    """rbacktransform / crbacktransform (numba_backend.py:326-375, :759-822) on
    random rotations, power-of-two segment scales, both modes, a zero column."""
    rng = np.random.default_rng(21)
    store = {}
    tags = []
    for n, b_r, b, cplx, mode, omega in ((70, 16, 4, False, 1, _DMAX / 2 / 16),
                                         (70, 16, 4, False, 0, 1e-3),
                                         (129, 32, 3, True, 1, _DMAX / 2 / 32),
                                         (129, 32, 3, True, 0, 1e-2),
                                         (40, 40, 2, False, 0, _DMAX / 2 / 40)):
        N = (n + b_r - 1) // b_r
        tile_ends = np.array([min((t + 1) * b_r, n) for t in range(N)], dtype=np.int64)
        th = rng.uniform(0, 2 * np.pi, (n, b))
        c = np.cos(th)
        s = np.sin(th)
        seg = -rng.integers(0, 300, (N, b)).astype(np.int32)
        alpha = np.ldexp(1.0, seg)
        x = rng.standard_normal((n, 2 * b if cplx else b)) * 10.0 ** rng.integers(-5, 5)
        if b >= 3:
            x[:, -1] = 0.0  # zero column: no normalisation / sweep (:347-350)
            if cplx:
                x[:, -2] = 0.0
        norms_out = np.zeros(b)
        alpha_out = np.zeros(b)
        xo = x.copy()
        if cplx:
            phi = rng.uniform(0, 2 * np.pi, (n, b))
            cre, cim = c * np.cos(phi), c * np.sin(phi)
            K.crbacktransform(cre, cim, s, alpha, tile_ends, xo, norms_out, alpha_out, mode, omega)
        else:
            cre, cim = c, np.zeros_like(c)
            K.rbacktransform(c, s, alpha, tile_ends, xo, norms_out, alpha_out, mode, omega)
        t = f"b{len(tags)}"
        store.update({f"{t}_meta": np.array([n, b_r, b, int(cplx), mode], dtype=np.int64),
                      f"{t}_omega": np.float64(omega), f"{t}_cre": cre, f"{t}_cim": cim,
                      f"{t}_s": s, f"{t}_seg": seg, f"{t}_x": x, f"{t}_xout": xo,
                      f"{t}_norms": norms_out, f"{t}_alpha": alpha_out})
        tags.append(t)
    save("backtransform", tags=np.array(tags), **store)


def _henry_case(store, tag, h, lam, b):
    """Henry's kernels as henry_rq_solve (reference.py:21-60) drives them: x and
    the packed status (0 = ok).  The kernels are called directly because the
    numba henry_solve_complex falls off its end on success (returns None, not
    0, K/numba_backend.py:876-923), which makes the public complex wrapper
    raise TypeError in unpack_status; the real wrapper is checked to agree."""
    from hessrq.reference import henry_rq_solve

    n = h.shape[0]
    lam_arr = np.atleast_1d(np.asarray(lam))
    cplx = np.iscomplexobj(lam_arr)
    m = lam_arr.shape[0]
    if cplx:
        x = np.ascontiguousarray(np.asarray(b, dtype=np.complex128).reshape(n, m)).copy()
        st = K.henry_solve_complex(np.asfortranarray(h), np.ascontiguousarray(lam_arr, dtype=np.complex128), x)
    else:
        x = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(n, m)).copy()
        st = K.henry_solve_real(np.asfortranarray(h), np.ascontiguousarray(lam_arr, dtype=np.float64), x)
        if st == 0:
            xr = henry_rq_solve(h, lam, b)
            assert np.array_equal(np.asarray(xr).reshape(n, m), x, equal_nan=True)
    st = 0 if st is None else int(st)
    store[f"{tag}_h"] = np.asfortranarray(h)
    store[f"{tag}_lam"] = np.asarray(lam)
    store[f"{tag}_b"] = np.asarray(b)
    store[f"{tag}_status"] = np.int64(st)
    if st == 0:
        store[f"{tag}_x"] = x


def gen_henry():
    """Henry's single sweep (K/numba_backend.py:830-923 via reference.py:21-60):
    random shifts, eigenvalue shifts (near-singular), n = 1/2, a scalar shift
    with a 1-D rhs, an overflowing rhs (unguarded: inf/nan propagate), an
    exactly singular integer system and a degenerate (zero subdiagonal) one."""
    rng = np.random.default_rng(41)
    store = {}
    tags = []

    def add(h, lam, b):
        t = f"y{len(tags)}"
        _henry_case(store, t, h, lam, b)
        tags.append(t)

    for n, m, seed in ((1, 2, 1), (2, 3, 2), (5, 3, 3), (40, 4, 4), (129, 5, 5), (300, 3, 6)):
        h = np.array(random_unreduced(n, seed).data)
        nrm = np.max(np.sum(np.abs(h), axis=1))
        add(h, nrm * rng.uniform(-2, 2, m), rng.standard_normal((n, m)))
        add(h, nrm * (rng.uniform(-2, 2, m) + 1j * rng.uniform(0.05, 2, m)),
            rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m)))
        if n >= 5:
            ev = np.linalg.eigvals(h)
            er, ec = ev[ev.imag == 0].real[:3], ev[ev.imag > 0][:3]
            if er.size:
                add(h, er, np.ones((n, er.size)))
            if ec.size:
                add(h, ec, np.ones((n, ec.size)) + 0j)
    h = np.array(random_unreduced(30, 9).data)
    add(h, 0.75, rng.standard_normal(30))                       # scalar shift, 1-D rhs
    add(h, 0.75 + 0.5j, rng.standard_normal(30) + 0j)
    add(np.array(gen_h2(60).data), np.array([2.0]), 1e290 * np.ones((60, 1)))
    add(np.array(gen_h2(60).data), np.array([2.0 + 0.5j]), 1e290 * np.ones((60, 1)) + 0j)
    # exactly singular: small-integer H with an integer eigenvalue
    for trial in range(5000):
        hi = np.triu(rng.integers(-2, 3, (8, 8))).astype(float)
        hi[np.arange(1, 8), np.arange(7)] = rng.choice([-2.0, -1.0, 1.0, 2.0], 7)
        ev = np.linalg.eigvals(hi)
        ints = [round(e.real) for e in ev if abs(e.imag) < 1e-12 and abs(e.real - round(e.real)) < 1e-12]
        if ints:
            lam = np.array([ints[0] + 0.25, float(ints[0]), ints[0] + 0.5])
            add(hi, lam, np.ones((8, 3)))
            add(hi, lam + 0j, np.ones((8, 3)) + 0j)
            break
    # singular final pivot: v[0] = c(h00 - lam) + s h01 cancels exactly (c = -s)
    h2 = np.array([[2.0, 1.0], [1.0, 2.0]])
    add(h2, np.array([0.5, 1.0, 3.0]), np.ones((2, 3)))
    add(h2, np.array([0.5 + 0.5j, 1.0 + 0j, 3.0 + 0j]), np.ones((2, 3)) + 0j)
    # degenerate rotation: a = h[n-1, n-2] = 0 and v[n-1] = h[n-1, n-1] - lam = 0
    hd = np.triu(rng.standard_normal((6, 6)), -1)
    hd[5, 4] = 0.0
    add(hd, np.array([0.3, hd[5, 5]]), np.ones((6, 2)))
    add(hd, np.array([0.3 + 0.1j, hd[5, 5] + 0j]), np.ones((6, 2)) + 0j)
    save("henry", tags=np.array(tags), **store)


def gen_hessenberg():
    """householder_hessenberg (testprob.py:146-174) on dense inputs: random
    matrices across the GPU panel width (64), an input that is already
    Hessenberg (returned unchanged with Q = I), a column that is already
    reduced mid-way (skip rule), graded rows, n = 1..3."""
    from hessrq.testprob import householder_hessenberg

    rng = np.random.default_rng(23)
    store = {}
    tags = []

    def add(a):
        hh, q = householder_hessenberg(a)
        t = f"d{len(tags)}"
        store[f"{t}_a"] = np.asfortranarray(a)
        store[f"{t}_h"] = np.asfortranarray(hh)
        store[f"{t}_q"] = np.asfortranarray(q)
        tags.append(t)

    for n in (1, 2, 3, 8, 50, 64, 65, 130, 200):
        add(rng.standard_normal((n, n)))
    add(np.array(random_unreduced(40, 2).data))
    a = rng.standard_normal((90, 90))
    a[12:, 10] = 0.0
    a[71:, 69] = 0.0
    add(a)
    d = np.ldexp(1.0, np.arange(100) // 5)
    add(rng.standard_normal((100, 100)) * d[:, None] / d[None, :])
    save("hessenberg", tags=np.array(tags), **store)


def gen_compact():
    """Stewart compact rotation codes (givens.py:90-198) through the
    reference's table functions (GivensTable.compact / from_compact,
    core.py:193-209): rotations built by make_real / make_complex from random
    and edge-case pairs, and raw codes across every window edge."""
    from hessrq import givens

    rng = np.random.default_rng(17)
    a = rng.standard_normal(3000) * np.ldexp(1.0, rng.integers(-40, 40, 3000))
    b = rng.standard_normal(3000) * np.ldexp(1.0, rng.integers(-40, 40, 3000))
    a[:10] = [0.0, 1.0, -1.0, 0.0, 0.0, 2.0, -2.0, 3.0, 1e-300, 5.0]
    b[:10] = [1.0, 0.0, 0.0, -1.0, 0.0, 2.0, 2.0, -3.0, 1.0, 1e-300]
    rots = [givens.make_real(x, y) for x, y in zip(a, b)]
    c = np.array([r.c for r in rots]).reshape(60, 50)
    s_ = np.array([r.s for r in rots]).reshape(60, 50)
    c[0, :6] = [-0.0, 0.0, -1.0, 1.0, 0.6, -0.6]
    s_[0, :6] = [1.0, -1.0, -0.0, 0.0, 0.8, -0.8]
    t = givens.compact_encode_table(c, s_)
    dc, ds = givens.compact_decode_table(t)
    v = (rng.standard_normal(3000) + 1j * rng.standard_normal(3000)) * np.ldexp(1.0, rng.integers(-30, 30, 3000))
    v[:4] = [0.0, 1j, -1.0, 1e-300 + 0j]
    a2 = a.copy()
    a2[:4] = [1.0, 0.0, 0.5, 0.0]
    crs = [givens.make_complex(x, y) for x, y in zip(a2, v)]
    cre = np.array([r.c.real for r in crs]).reshape(60, 50)
    cim = np.array([r.c.imag for r in crs]).reshape(60, 50)
    cs = np.array([r.s for r in crs]).reshape(60, 50)
    packed = givens.compact_encode_table_complex(cre, cim, cs)
    dre, dim, dcs = givens.compact_decode_table_complex(packed)
    codes = np.concatenate([rng.uniform(-7, 7, 2000),
                            [0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 3.0, -3.0, 4.0, -4.0, 5.0, -5.0,
                             6.0, -6.0, 7.0, -7.0, np.nextafter(1.0, 2.0), np.nextafter(3.0, 4.0),
                             np.nextafter(5.0, 6.0), 2.5, -6.25]])
    kc, ks = givens.compact_decode_table(codes)
    save("compact", c=c, s=s_, t=t, dc=dc, ds=ds, cre=cre, cim=cim, cs=cs, packed=packed,
         dre=dre, dim=dim, dcs=dcs, codes=codes, kc=kc, ks=ks)


def gen_runstats():
    """RunStats flops / formula per task type of reference solves (the bench
    CSV's flops_* and formula_* columns, cli.py:320-364)."""
    from hessrq.scheduler import RunStats

    store = {}
    tags = []
    for n, b_r, m, cplx in ((300, 64, 3, False), (300, 64, 3, True), (129, 32, 2, True),
                            (200, 200, 2, False)):
        h = random_unreduced(n, 3)
        lam = np.linspace(0.5, 1.5, m) * h.infinity_norm() * 2 + (0.3j if cplx else 0)
        b = np.ones((n, m), dtype=complex if cplx else float)
        st = RunStats()
        (chsrq3 if cplx else dhsrq3)(h, lam, b, b_r=b_r, b_c=8, stats=st)
        t = f"r{len(tags)}"
        store[f"{t}_meta"] = np.array([n, b_r, m, int(cplx)], dtype=np.int64)
        store[f"{t}_flops"] = np.array([st.flops.get(k, 0.0) for k in
                                        ("ReduceDiag", "ReduceOffdiag", "Solve", "Update", "Backtransform")])
        store[f"{t}_formula"] = np.array([st.formula.get(k, 0.0) for k in
                                          ("ReduceDiag", "ReduceOffdiag", "Solve", "Update", "Backtransform")])
        tags.append(t)
    # the bench command's shift generator and CSV header (cli.py:79-95, 320-331)
    from hessrq import cli

    hb = random_unreduced(50, 4)
    store["shifts_real"] = cli.load_shifts("gen:count=7,kind=real,seed=2,radius=1.5", hb)
    store["shifts_cplx"] = cli.load_shifts("gen:count=7,kind=complex,seed=2,radius=1.5", hb)
    store["shifts_h"] = np.asfortranarray(hb.data)
    store["bench_header"] = np.array(
        ["schema", "backend", "n", "m", "kind", "b_r", "b_c", "workers", "robust"]
        + list(cli.TASK_TYPES) + ["total_s"] + [f"flops_{t}" for t in cli.TASK_TYPES]
        + [f"formula_{t}" for t in cli.TASK_TYPES] + ["henry_s"])
    save("runstats", tags=np.array(tags), **store)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected fixtures: make_golden.py henry tiles ...
        for name in sys.argv[1:]:
            globals()[f"gen_{name}"]()
        sys.exit(0)
    gen_hessenberg()
    gen_compact()
    gen_runstats()
    gen_henry()
    gen_backtransform()
    gen_singular()
    gen_scalars()
    gen_tiles()
    gen_solves()
    gen_inviter()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
