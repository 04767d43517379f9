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
