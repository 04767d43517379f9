"""GPU parity on the BASELINE.json instances and on exactly singular shifts.

* singular: small-integer matrices with an exact eigenvalue (golden
  fixtures from the live reference, tools/make_golden.py gen_singular): in
  one tile the GPU raises SingularSystemError with the reference's
  shift_index and local_index; across tiles see the test's docstring.
* configs 3/4/5 (H bit-reproducible from the seed, shifts = the committed
  LAPACK eigenvalues under data/): a seeded sample of each selection solved on
  the GPU at the config's full n and b_r = 128 and compared with the CPU
  oracle on the same start vector -- segment exponents exact in every tile but
  tile 0 (+-1, the rounding-level final pivot), vectors phase-aligned to
  1e-8 (north_star), residual ||Hx - lx|| / (||H||_F ||x||) <= 10 n eps.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _align(x, ref):
    ip = np.vdot(x, ref)
    return x * (ip / abs(ip)) if ip != 0 else x


def test_singular_shifts_raise_like_reference(dev):
    """Exact-zero pivots of exactly singular systems.

    Within one tile (b_r >= n) the GPU performs the reference's arithmetic
    bit for bit, so the zero pivot -- and the error, with its shift_index and
    local_index -- is reproduced exactly.  Across tiles the crossover column
    comes from the panel GEMM (a different summation order than the
    reference's rotation-by-rotation recursion), so the rounding-level final
    pivot need not land on exactly 0.0: then the GPU must either raise the
    same error or return a finite result, and the inverse-iteration driver
    a converged eigenvector with residual <= 10 n eps.
    """
    from paper_2101_05063_b200 import (InviterConfig, SingularSystemError, TaskError, chsrq3,
                                       dhsrq3, hsrq3in)

    g = golden("singular")
    kinds = [str(k) for k in g["node_kinds"]]
    exact = 0
    for t in g["tags"]:
        h, lam = g[f"{t}_h"], g[f"{t}_lam"]
        cplx = bool(int(g[f"{t}_cplx"]))
        n = h.shape[0]
        b = np.ones((n, lam.size)) + (0j if cplx else 0)
        f = chsrq3 if cplx else dhsrq3
        for (b_r, b_c, shift, row), node, msg in zip(g[f"{t}_hits"], g[f"{t}_nodes"],
                                                     g[f"{t}_messages"]):
            if b_r >= n:
                with pytest.raises(SingularSystemError) as e:
                    f(h, lam, b, b_r=int(b_r), b_c=int(b_c))
                assert (e.value.shift_index, e.value.local_index) == (shift, row)
                # ... raised as the reference's caller sees it: the executor's
                # TaskError naming the failing node (scheduler.py:182-187)
                err = e.value
                assert isinstance(err, TaskError) and err.__cause__ is err.cause
                assert err.node.kind == kinds[node[0]]
                assert tuple(err.node.coords) == tuple(int(v) for v in node[1:4])
                assert err.node.seq == node[4] and str(err) == str(msg)
                exact += 1
                continue
            try:
                r = f(h, lam, b, b_r=int(b_r), b_c=int(b_c))
            except SingularSystemError as e:
                assert (e.shift_index, e.local_index) == (shift, row)
            else:
                assert np.all(np.isfinite(r.x))
        want = g[f"{t}_inviter"]
        z = lam[1]
        try:
            r = hsrq3in(h, np.array([z]), InviterConfig(b_r=3, b_c=2))
        except SingularSystemError as e:
            assert (e.shift_index, e.local_index) == tuple(want)
        else:
            x = r.vectors[:, 0]
            eps = np.finfo(float).eps
            assert r.converged[0]
            assert np.linalg.norm(h @ x - z * x) / (np.linalg.norm(h, "fro") * np.linalg.norm(x)) <= 10 * n * eps
    assert exact >= 4


def _sample(cfg, nr, nc, seed):
    import instances

    sel = instances.shifts(cfg)
    rng = np.random.default_rng(100 + cfg + seed)
    er = sel[sel.imag == 0].real
    ec = sel[sel.imag > 0]
    er = er[rng.choice(er.size, min(nr, er.size), replace=False)] if er.size else er
    ec = ec[rng.choice(ec.size, min(nc, ec.size), replace=False)] if ec.size else ec
    return instances.make_h(cfg), er, ec


@pytest.mark.parametrize("cfg,nr,nc", [(3, 0, 8), (4, 6, 6), (5, 4, 4)])
def test_config_sample_matches_oracle(dev, oracle, cfg, nr, nc):
    from paper_2101_05063_b200 import solver

    h, er, ec = _sample(cfg, nr, nc, 0)
    n = h.shape[0]
    b_r = 128
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = rho * np.ones(n)
    out, _ = solver.solve_group(h, ec, er, start, b_r)
    assert out.nfail == 0
    X = out.X.cpu().numpy()
    seg = out.seg_exp.cpu().numpy()
    mc = ec.size
    threads = os.cpu_count() or 1
    parts = []
    if mc:
        parts.append(oracle.solve(h, ec, np.repeat(start[:, None], mc, 1).astype(complex), b_r,
                                  b_c=1, mode="eigvec", nthreads=threads))
    if er.size:
        parts.append(oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, b_c=1,
                                  mode="eigvec", nthreads=threads))
    want = np.concatenate([p.segment_exp for p in parts], axis=1)
    assert np.array_equal(seg[1:], want[1:])
    assert np.max(np.abs(seg[0] - want[0])) <= 1
    hf = np.linalg.norm(h, "fro")
    eps = np.finfo(float).eps
    refs = np.concatenate([p.x for p in parts], axis=1)
    lams = np.concatenate([ec, er.astype(complex)])
    l2 = out.log2norm.cpu().numpy()
    l2w = np.concatenate([p.log2norm for p in parts])
    for l in range(lams.size):
        x = X[2 * l] + 1j * X[2 * l + 1] if l < mc else X[2 * mc + (l - mc)].astype(complex)
        ref = refs[:, l]
        assert np.linalg.norm(_align(x, ref) - ref) <= 1e-8, l
        assert np.linalg.norm(h @ x - lams[l] * x) / (hf * np.linalg.norm(x)) <= 10 * n * eps, l
    assert np.all(np.abs(l2 - l2w) < 4.0)
    # both sides agree on convergence (inviter.py:71-73)
    assert np.array_equal(solver.converged_log2(l2, n), solver.converged_log2(l2w, n))


def _oracle_excluding_singular(oracle, h, lam, start, b_r, threads):
    """Oracle solve of ``lam`` (one reference call per shift batch of 1); an
    exactly singular shift raises in the reference (backsolve.py:53-59) --
    it is recorded and excluded, and the rest re-solved."""
    keep = np.arange(lam.size)
    singular = []
    while True:
        b = np.repeat(start[:, None], keep.size, 1)
        try:
            return oracle.solve(h, lam[keep], b.astype(lam.dtype), b_r, b_c=1, mode="eigvec",
                                nthreads=threads), keep, singular
        except oracle.OracleError as e:
            assert e.phase == 2, "only singular factors are expected"
            singular.append(int(keep[e.shift_index]))
            keep = np.delete(keep, e.shift_index)


def test_config2_all_shifts_match_oracle(dev, oracle):
    """Config 2 (BASELINE.json): n = 4000, lambda_i = i/n + 1, every 4th real
    eigenvalue (1000 shifts), b_r = 64 with a ragged last tile (4000 = 62*64 +
    32), through dhsrq3in's seam (inviter.py:155-161).  H is rebuilt on this
    box (LAPACK's Hessenberg reduction is reproducible only to rounding), the
    shifts are this container's cached eigenvalues.  All 1000 shifts against
    the oracle on the same H; an exactly singular shift (the reference raises)
    must either raise with the same shift index on the GPU or return a
    finite, converged vector (the GEMM-form crossover rounds the final pivot
    differently across tiles)."""
    import instances
    from paper_2101_05063_b200 import SingularSystemError, solver

    h = instances.make_h(2)
    lam = instances.shifts(2)
    n, b_r = h.shape[0], 64
    assert lam.size == 1000 and n % b_r == 32
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = rho * np.ones(n)
    o, keep, singular = _oracle_excluding_singular(oracle, h, lam, start, b_r, os.cpu_count() or 1)
    try:
        out, _ = solver.solve_group(h, [], lam, start, b_r)
        fails = out.fail.cpu().numpy()
    except SingularSystemError as e:  # pragma: no cover - instance dependent
        assert e.shift_index in singular
        return
    bad = set(np.nonzero(fails)[0].tolist())
    assert bad <= set(singular), (bad, singular)
    X = out.X.cpu().numpy()
    seg = out.seg_exp.cpu().numpy()
    assert np.array_equal(seg[1:, keep], o.segment_exp[1:])
    assert np.max(np.abs(seg[0, keep] - o.segment_exp[0])) <= 1
    err = max(np.linalg.norm(_align(X[q], o.x[:, i]) - o.x[:, i]) for i, q in enumerate(keep))
    assert err <= 1e-8, err
    hf = np.linalg.norm(h, "fro")
    R = h @ X.T - X.T * lam[None, :]
    res = np.linalg.norm(R, axis=0) / (hf * np.linalg.norm(X, axis=1))
    ok = np.setdiff1d(np.arange(lam.size), list(bad))
    assert np.all(res[ok] <= 10 * n * np.finfo(float).eps), res.max()
    l2 = out.log2norm.cpu().numpy()
    assert np.all(np.abs(l2[keep] - o.log2norm) < 4.0)
    assert np.array_equal(solver.converged_log2(l2[keep], n), solver.converged_log2(o.log2norm, n))


def test_config5_all_shifts_residual_and_stratified_oracle(dev, oracle):
    """Config 5 at full size: n = 16000, all 3790 real + 6105 complex shifts
    (north_star: "oracle-matching eigenvectors for n=16000 with all shifts"),
    b_r = 128, through solver.solve_group -- the production seam with the
    automatically selected kernel variants (warp-pair complex sweep at DP 4,
    backtransform G = 8).  Every column: converged (inviter.py:71-73) and
    ||Hx - lx|| / (||H||_F ||x||) <= 10 n eps (checked with a torch fp64 GEMM
    on the device: test infrastructure).  A stratified sample of 40 real + 40
    complex shifts (evenly spaced along each kind's sorted spectrum) against
    the oracle on the same start vector."""
    import instances
    from paper_2101_05063_b200 import solver

    h = instances.make_h(5)
    sel = instances.shifts(5)
    er = sel[sel.imag == 0].real
    ec = sel[sel.imag > 0]
    assert (er.size, ec.size) == (3790, 6105)
    n, b_r = h.shape[0], 128
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = rho * np.ones(n)
    out, gs = solver.solve_group(h, ec, er, start, b_r)
    assert out.nfail == 0
    mc = ec.size
    l2 = out.log2norm.cpu().numpy()
    assert np.all(solver.converged_log2(l2, n)), int(np.count_nonzero(~solver.converged_log2(l2, n)))
    # residuals of all 16000 columns on the device
    Hd = torch.from_numpy(np.ascontiguousarray(h)).to(dev)
    X = out.X  # (ncol, n): row c = column c
    HX = torch.matmul(Hd, X.T)  # (n, ncol)
    lre = torch.from_numpy(np.concatenate([ec.real, er])).to(dev)
    lim = torch.from_numpy(ec.imag).to(dev)
    R = HX.T.clone()  # (ncol, n)
    R[2 * mc:] -= lre[mc:, None] * X[2 * mc:]
    xr, xi = X[0:2 * mc:2], X[1:2 * mc:2]
    R[0:2 * mc:2] -= lre[:mc, None] * xr - lim[:, None] * xi
    R[1:2 * mc:2] -= lre[:mc, None] * xi + lim[:, None] * xr
    rn2 = (R * R).sum(1)
    xn2 = (X * X).sum(1)
    rn = torch.cat([(rn2[0:2 * mc:2] + rn2[1:2 * mc:2]).sqrt(), rn2[2 * mc:].sqrt()])
    xn = torch.cat([(xn2[0:2 * mc:2] + xn2[1:2 * mc:2]).sqrt(), xn2[2 * mc:].sqrt()])
    res = (rn / (torch.linalg.norm(Hd) * xn)).cpu().numpy()
    del Hd, HX, R
    eps = np.finfo(float).eps
    assert res.size == 9895 and np.all(res <= 10 * n * eps), (res.max() / (n * eps), int(res.argmax()))
    # stratified oracle sample
    ir = np.linspace(0, er.size - 1, 40).round().astype(int)
    ic = np.linspace(0, ec.size - 1, 40).round().astype(int)
    order_r, order_c = np.argsort(er), np.argsort(ec.real)
    ir, ic = order_r[ir], order_c[ic]
    threads = os.cpu_count() or 1
    o_r = oracle.solve(h, er[ir], np.repeat(start[:, None], ir.size, 1), b_r, b_c=1,
                       mode="eigvec", nthreads=threads)
    o_c = oracle.solve(h, ec[ic], np.repeat(start[:, None], ic.size, 1).astype(complex), b_r,
                       b_c=1, mode="eigvec", nthreads=threads)
    seg = out.seg_exp.cpu().numpy()
    Xh = {}
    for name, idx, o, off in (("c", ic, o_c, 0), ("r", ir, o_r, mc)):
        q = off + idx
        assert np.array_equal(seg[1:, q], o.segment_exp[1:]), name
        assert np.max(np.abs(seg[0, q] - o.segment_exp[0])) <= 1, name
        assert np.all(np.abs(l2[q] - o.log2norm) < 4.0), name
        for i, qq in enumerate(idx):
            if name == "c":
                x = (X[2 * qq] + 1j * X[2 * qq + 1]).cpu().numpy()
            else:
                x = X[2 * mc + qq].cpu().numpy()
            ref = o.x[:, i]
            d = np.linalg.norm(_align(x, ref) - ref)
            assert d <= 1e-8, (name, int(qq), d)
            Xh[(name, int(qq))] = d
    assert len(Xh) == 80


@pytest.mark.parametrize("cfg", [3, 4])
def test_config34_all_shifts_match_oracle(dev, oracle, cfg):
    """Configs 3 (n = 4000, all 1430 complex shifts Im > 0) and 4 (n = 2000
    graded, 602 real + 699 complex shifts perturbed by 1e-14) in full, b_r =
    128, one sweep of every shift vs the oracle on the same start vector:
    segment exponents exact (tile 0 +-1), vectors phase-aligned to 1e-8,
    residual <= 10 n eps on every column, the same convergence decisions."""
    import instances
    from paper_2101_05063_b200 import solver

    h = instances.make_h(cfg)
    sel = instances.shifts(cfg)
    er = sel[sel.imag == 0].real
    ec = sel[sel.imag > 0]
    n, b_r = h.shape[0], 128
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = rho * np.ones(n)
    out, _ = solver.solve_group(h, ec, er, start, b_r)
    assert out.nfail == 0
    threads = os.cpu_count() or 1
    parts = []
    if ec.size:
        parts.append(oracle.solve(h, ec, np.repeat(start[:, None], ec.size, 1).astype(complex), b_r,
                                  b_c=8, mode="eigvec", nthreads=threads))
    if er.size:
        parts.append(oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, b_c=8,
                                  mode="eigvec", nthreads=threads))
    want = np.concatenate([p.segment_exp for p in parts], axis=1)
    seg = out.seg_exp.cpu().numpy()
    assert np.array_equal(seg[1:], want[1:])
    assert np.max(np.abs(seg[0] - want[0])) <= 1
    X = out.X.cpu().numpy()
    mc = ec.size
    refs = np.concatenate([p.x for p in parts], axis=1)
    lams = np.concatenate([ec, er.astype(complex)])
    V = np.empty((n, lams.size), dtype=complex)
    V[:, :mc] = (X[0:2 * mc:2] + 1j * X[1:2 * mc:2]).T
    V[:, mc:] = X[2 * mc:].T
    ip = np.sum(V.conj() * refs, axis=0)
    ph = np.where(ip != 0, ip / np.abs(ip), 1.0)
    dev_err = np.linalg.norm(V * ph[None, :] - refs, axis=0)
    assert dev_err.max() <= 1e-8, (dev_err.max(), int(dev_err.argmax()))
    hf = np.linalg.norm(h, "fro")
    res = np.linalg.norm(h @ V - V * lams[None, :], axis=0) / (hf * np.linalg.norm(V, axis=0))
    assert res.max() <= 10 * n * np.finfo(float).eps, res.max()
    l2 = out.log2norm.cpu().numpy()
    l2w = np.concatenate([p.log2norm for p in parts])
    assert np.array_equal(solver.converged_log2(l2, n), solver.converged_log2(l2w, n))
