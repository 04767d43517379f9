"""The warp-specialised diagonal sweeps (k_diag_real_ws / k_diag_cplx_ws, a warp pair
per group of shifts: pivot chain beside the previous step's row update) give
bit-identical results to the one-warp sweeps (k_diag_real / k_diag_cplx), which the other
parity tests pin to the oracle -- on cases that take the guards' rescaling
and exact-certification paths, at every supported lanes-per-shift."""

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


@pytest.fixture
def lib(dev):
    from paper_2101_05063_b200 import _lib

    L = _lib.load()
    L.hsrq_tune_diag_rx(0)  # the one-warp sweeps are the reference here
    yield L
    L.hsrq_tune_diag(0, 0, 0, -1, -1)  # back to the automatic choice
    L.hsrq_tune_diag_rx(-1)


def _outputs(gs):
    return [t.cpu().numpy().copy() for t in (gs.X, gs.seg_exp, gs.alpha_exp, gs.norms, gs.c_re,
                                              gs.c_im, gs.s, gs.fail)]


@pytest.mark.parametrize("n,b_r,seed,kind,mode", [
    (700, 128, 3, "start", "eigvec"),
    (515, 100, 2, "huge", "eigvec"),
    (640, 128, 4, "rhs", "solve"),
    (600, 128, 5, "graded", "eigvec"),
    (301, 37, 6, "start", "eigvec"),
    (900, 128, 7, "realonly", "eigvec"),
])
@pytest.mark.parametrize("dp,ws", [(4, 2), (4, 3), (8, 2), (8, 4), (16, 2), (32, 4)])
def test_ws_sweep_matches_one_warp_sweep(dev, lib, n, b_r, seed, kind, mode, dp, ws):
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h = (instances.graded_hessenberg if kind == "graded" else instances.random_hessenberg)(n, seed)
    ev = np.linalg.eigvals(h)
    er = ev[ev.imag == 0].real[:7]
    ec = ev[ev.imag > 0][:45]
    if kind == "realonly":  # a group without complex shifts
        er = np.concatenate([ev[ev.imag == 0].real, ev[ev.imag > 0].real[:30] + 1e-3])
        ec = ec[:0]
    rng = np.random.default_rng(seed)
    if kind == "rhs":
        er, ec = er + 0.125, ec + 0.125j
        B = torch.from_numpy(rng.standard_normal((2 * ec.size + er.size, n))).to(dev)
    else:
        rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
        B = torch.full((n,), 1e300 if kind == "huge" else rho, dtype=torch.float64, device=dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    res = {}
    for w in (0, ws):
        lib.hsrq_tune_diag(dp, 4, 2 if dp == 4 else 4, w, w)
        gs = GroupSolver(dh, b_r, ec.size, er.size)
        gs.set_shifts(ec, er)
        nf = gs.launch(B, B.dim() == 1, mode=mode)
        res[w] = (nf, _outputs(gs))
    assert res[0][0] == res[ws][0]
    for a, b in zip(res[0][1], res[ws][1]):
        assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("n,b_r,seed,kind,mode", [
    (700, 128, 3, "start", "eigvec"),
    (515, 100, 2, "huge", "eigvec"),
    (640, 128, 4, "rhs", "solve"),
    (600, 128, 5, "graded", "eigvec"),
    (301, 37, 6, "start", "eigvec"),
])
@pytest.mark.parametrize("dp,np_rx", [(32, 4), (32, 8), (16, 4), (16, 8)])
def test_rx_sweep_matches_one_warp_sweep(dev, lib, n, b_r, seed, kind, mode, dp, np_rx):
    """k_diag_cplx_rx (rotation chain one step ahead of the solution chain,
    hsrq_diag_rx.cuh) vs k_diag_cplx at 16 and 32 lanes per shift: bitwise."""
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h = (instances.graded_hessenberg if kind == "graded" else instances.random_hessenberg)(n, seed)
    ev = np.linalg.eigvals(h)
    er = ev[ev.imag == 0].real[:7]
    ec = ev[ev.imag > 0][:45]
    rng = np.random.default_rng(seed)
    if kind == "rhs":
        er, ec = er + 0.125, ec + 0.125j
        B = torch.from_numpy(rng.standard_normal((2 * ec.size + er.size, n))).to(dev)
    else:
        rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
        B = torch.full((n,), 1e300 if kind == "huge" else rho, dtype=torch.float64, device=dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    res = {}
    try:
        for rx in (0, np_rx):
            lib.hsrq_tune_diag(dp, 16, 16, 0, 0)
            lib.hsrq_tune_diag_rx(rx)
            gs = GroupSolver(dh, b_r, ec.size, er.size)
            gs.set_shifts(ec, er)
            nf = gs.launch(B, B.dim() == 1, mode=mode)
            res[rx] = (nf, _outputs(gs))
    finally:
        lib.hsrq_tune_diag_rx(-1)
    assert res[0][0] == res[np_rx][0]
    for a, b in zip(res[0][1], res[np_rx][1]):
        assert np.array_equal(a, b, equal_nan=True)
