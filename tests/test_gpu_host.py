"""hsrq_solve_group_host (host buffers, H streamed in column blocks overlapped
with the sweep) returns exactly what the device-buffer entry point returns."""

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


@pytest.mark.parametrize("n,b_r,seed,kind,robust,mode", [
    (300, 37, 1, "start", True, "eigvec"),
    (515, 100, 2, "huge", True, "eigvec"),
    (1000, 128, 3, "start", True, "eigvec"),
    (640, 128, 4, "rhs", True, "solve"),
    (200, 16, 5, "rhs", False, "solve"),
])
def test_host_entry_matches_device_entry(dev, n, b_r, seed, kind, robust, mode):
    import instances
    from paper_2101_05063_b200 import solver

    h = instances.random_hessenberg(n, seed)
    ev = np.linalg.eigvals(h)
    rng = np.random.default_rng(seed)
    er = ev[ev.imag == 0].real[:5]
    ec = ev[ev.imag > 0][:6]
    if kind == "rhs":
        er = er + 0.125
        ec = ec + 0.125j
    ncol = 2 * ec.size + er.size
    if kind == "rhs":
        b = rng.standard_normal((ncol, n))
    else:
        rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
        b = (rho if kind == "start" else 1e300) * np.ones(n)
    dout, _ = solver.solve_group(h, ec, er, torch.from_numpy(b), b_r, robust=robust, mode=mode)
    hout = solver.solve_group_host(h, ec, er, b, b_r, robust=robust, mode=mode)
    assert hout.nfail == dout.nfail
    assert np.array_equal(hout.X, dout.X.cpu().numpy())
    assert np.array_equal(hout.seg_exp, dout.seg_exp.cpu().numpy())
    assert np.array_equal(hout.alpha_exp, dout.alpha_exp.cpu().numpy())
    assert np.array_equal(hout.norms, dout.norms.cpu().numpy(), equal_nan=True)
    assert np.array_equal(hout.log2norm, dout.log2norm.cpu().numpy(), equal_nan=True)
    assert np.array_equal(hout.fail, dout.fail.cpu().numpy())
