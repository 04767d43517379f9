"""GPU vs CPU oracle where the overflow guards actually fire.

Random unreduced Hessenberg matrices (BASELINE config 3 construction) with
eigenvalue shifts grow the solution by 2^hundreds, so every ProtectUpdate
step and the segment-scale bookkeeping is exercised, for real and complex
shifts, full and ragged tiles, several b_r.  Scale exponents must agree
exactly; vectors after phase alignment to 1e-8 (north_star); every vector
must satisfy the residual bound ||Hx - lx|| / (||H||_F ||x||) <= 10 n eps.
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _align(x, ref):
    ip = np.vdot(x, ref)
    return x * (ip / abs(ip)) if ip != 0 else x


def _case(n, seed, nr, nc):
    import instances

    h = instances.random_hessenberg(n, seed)
    ev = np.linalg.eigvals(h)
    rng = np.random.default_rng(seed)
    er = ev[ev.imag == 0].real
    ec = ev[ev.imag > 0]
    er = er[rng.choice(er.size, min(nr, er.size), replace=False)]
    ec = ec[rng.choice(ec.size, min(nc, ec.size), replace=False)]
    return h, er, ec


@pytest.mark.parametrize("n,b_r,seed,rhs", [
    (1000, 128, 0, 1.0), (700, 64, 1, 1.0), (515, 100, 2, 1.0), (300, 37, 3, 1.0),
    (1000, 128, 4, 1e300), (700, 64, 5, 1e300), (515, 100, 6, 1e300), (300, 37, 7, 1e300),
    (256, 32, 8, 1e300), (128, 16, 9, 1e300)])
def test_scaling_matches_oracle(dev, oracle, n, b_r, seed, rhs):
    """rhs = 1: the start vector eps*||H||*ones; rhs = 1e300: a start vector near
    overflow, so every guard (solve, steps 1-3, backtransform) must fire."""
    from paper_2101_05063_b200 import solver

    h, er, ec = _case(n, seed, 6, 6)
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = (rho if rhs == 1.0 else rhs) * np.ones(n)
    out, _ = solver.solve_group(h, ec, er, start, b_r)
    assert out.nfail == 0
    X = out.X.cpu().numpy()
    seg = out.seg_exp.cpu().numpy()
    mc = ec.size
    o_c = oracle.solve(h, ec, np.repeat(start[:, None], mc, 1).astype(complex), b_r, mode="eigvec")
    o_r = oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, mode="eigvec")
    if rhs > 1.0:  # the guards fired (otherwise this case would not test scaling)
        assert seg.min() < 0 and o_r.segment_exp.min() < 0
    # Scale exponents are exact in every tile but the first: tile 0 holds the
    # final pivot, which for an eigenvalue shift is rounding-level, so its
    # guard (numba_backend.py:184-191) may land one power of two apart when
    # the crossover summation order differs (the GEMM-form reduction).
    want = np.concatenate([o_c.segment_exp, o_r.segment_exp], axis=1)
    assert np.array_equal(seg[1:], want[1:])
    assert np.max(np.abs(seg[0] - want[0])) <= 1
    da = out.alpha_exp.cpu().numpy() - np.concatenate([o_c.alpha_exp, o_r.alpha_exp])
    assert np.max(np.abs(da)) <= 1
    hf = np.linalg.norm(h, "fro")
    eps = np.finfo(float).eps
    for l in range(mc):
        x = X[2 * l] + 1j * X[2 * l + 1]
        assert np.linalg.norm(_align(x, o_c.x[:, l]) - o_c.x[:, l]) <= 1e-8
        assert np.linalg.norm(h @ x - ec[l] * x) / (hf * np.linalg.norm(x)) <= 10 * n * eps
    for l in range(er.size):
        x = X[2 * mc + l]
        assert np.linalg.norm(_align(x, o_r.x[:, l]) - o_r.x[:, l]) <= 1e-8
        assert np.linalg.norm(h @ x - er[l] * x) / (hf * np.linalg.norm(x)) <= 10 * n * eps
    # Represented norms ~ 1/(last pivot); with eigenvalue shifts the pivot is
    # rounding-level, so only its order of magnitude is reproducible across
    # summation orders (observed |d log2| <= 0.7); both pass the convergence test.
    l2 = out.log2norm.cpu().numpy()
    assert np.all(np.abs(l2 - np.concatenate([o_c.log2norm, o_r.log2norm])) < 4.0)


def test_lookahead_is_bitwise_neutral(monkeypatch):
    """The lookahead schedule (diag sweep of column jt-1 beside the rest of
    panel jt, double-buffered panel operands) changes the order of execution
    only: results are bit-identical to the serial schedule, across the diag
    kernel variants the shift count selects."""
    from paper_2101_05063_b200.solver import solve_group

    rng = np.random.default_rng(4)
    n, b_r = 900, 128
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    er = rng.uniform(-3, 3, 40)
    ec = rng.uniform(-3, 3, 33) + 1j * rng.uniform(0.1, 2, 33)
    b = np.full(n, 1e300)  # every guard path fires
    outs = []
    for la in ("0", "1"):
        monkeypatch.setenv("HSRQ_LOOKAHEAD", la)
        out, _ = solve_group(h, ec, er, b, b_r)
        outs.append((out.X.cpu().numpy().copy(), out.seg_exp.cpu().numpy().copy(),
                     out.norms.cpu().numpy().copy(), out.nfail))
    (x0, s0, n0, f0), (x1, s1, n1, f1) = outs
    assert f0 == f1 == 0
    assert np.array_equal(x0.view(np.int64), x1.view(np.int64))
    assert np.array_equal(s0, s1) and np.array_equal(n0.view(np.int64), n1.view(np.int64))
