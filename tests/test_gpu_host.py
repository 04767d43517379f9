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


def test_async_host_entry_two_in_flight(dev):
    """hsrq_solve_group_host_async: three different solve groups enqueued
    back to back on two workspaces (the third reuses the first after waiting)
    give exactly the synchronous entry's results."""
    import instances
    from paper_2101_05063_b200.solver import HostGroupSolver

    n, b_r = 700, 128
    h = np.asfortranarray(instances.random_hessenberg(n, 9))
    ev = np.linalg.eigvals(h)
    groups = []
    for off in (0.0, 0.25, 0.5):
        er = ev[ev.imag == 0].real[:4] + off
        ec = ev[ev.imag > 0][:5] + 1j * off
        lam = np.concatenate([ec, er.astype(np.complex128)])
        groups.append((np.ascontiguousarray(lam.real), np.ascontiguousarray(lam.imag)))
    b = np.full(n, 1e-3)
    solvers = [HostGroupSolver(n, b_r, 5, 4, dev), HostGroupSolver(n, b_r, 5, 4, dev)]
    want = []
    for lre, lim in groups:
        o = solvers[0].new_output()
        want.append(solvers[0].launch(h, lre, lim, b, True, o))
    outs = [solvers[0].new_output(pinned=True), solvers[1].new_output(pinned=True)]
    got = []
    t0 = solvers[0].launch(h, *groups[0], b, True, outs[0], wait=False)
    t1 = solvers[1].launch(h, *groups[1], b, True, outs[1], wait=False)
    solvers[0].wait_ticket(t0, outs[0])
    got.append((outs[0].X.copy(), outs[0].seg_exp.copy(), outs[0].nfail))
    t2 = solvers[0].launch(h, *groups[2], b, True, outs[0], wait=False)
    solvers[1].wait_ticket(t1, outs[1])
    got.append((outs[1].X.copy(), outs[1].seg_exp.copy(), outs[1].nfail))
    solvers[0].wait_ticket(t2, outs[0])
    got.append((outs[0].X.copy(), outs[0].seg_exp.copy(), outs[0].nfail))
    for w, (x, seg, nf) in zip(want, got):
        assert nf == w.nfail
        assert np.array_equal(x, w.X) and np.array_equal(seg, w.seg_exp)


def test_graph_replay_matches_eager(dev):
    """hsrq_graph_capture / hsrq_graph_launch: a captured solve replays the
    eager solve bit for bit, and picks up new shifts written into the same
    buffers (GroupSolver.set_shifts) between replays."""
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    n, b_r = 640, 64
    h = instances.random_hessenberg(n, 12)
    ev = np.linalg.eigvals(h)
    er, ec = ev[ev.imag == 0].real[:6], ev[ev.imag > 0][:5]
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    b = torch.full((n,), 1e-3, dtype=torch.float64, device=dev)
    gs = GroupSolver(dh, b_r, ec.size, er.size)
    gs.set_shifts(ec, er)
    gs.capture(b, True)
    results = []
    for off in (0.0, 0.125):
        gs.set_shifts(ec + 1j * off, er + off)
        nf = gs.replay()
        results.append((nf, gs.X.cpu().numpy().copy(), gs.seg_exp.cpu().numpy().copy()))
    ref = GroupSolver(dh, b_r, ec.size, er.size)
    for (nf, X, seg), off in zip(results, (0.0, 0.125)):
        ref.set_shifts(ec + 1j * off, er + off)
        rnf = ref.launch(b, True)
        assert nf == rnf
        assert np.array_equal(X, ref.X.cpu().numpy()) and np.array_equal(seg, ref.seg_exp.cpu().numpy())


def test_sorted_shift_order_is_transparent(dev):
    """solve_group runs complex shifts sorted by imaginary part and puts every
    per-shift output back in the caller's order: identical to a GroupSolver
    launch with the caller's order, in both the broadcast and explicit-rhs
    forms."""
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver, solve_group

    n, b_r = 500, 64
    h = instances.random_hessenberg(n, 21)
    ev = np.linalg.eigvals(h)
    er, ec = ev[ev.imag == 0].real[:5], ev[ev.imag > 0][:9]
    ec = ec[np.argsort(-ec.imag)]  # deliberately not in sorted order
    rng = np.random.default_rng(0)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    for B in (np.full(n, 1e-3), rng.standard_normal((2 * ec.size + er.size, n))):
        out, _ = solve_group(h, ec, er, torch.from_numpy(B), b_r, mode="solve")
        ref = GroupSolver(dh, b_r, ec.size, er.size)
        ref.set_shifts(ec, er)
        ref.launch(torch.from_numpy(B).to(dev), B.ndim == 1, mode="solve")
        for a, r in ((out.X, ref.X), (out.seg_exp, ref.seg_exp), (out.norms, ref.norms),
                     (out.c_re, ref.c_re), (out.c_im, ref.c_im), (out.s, ref.s),
                     (out.alpha_exp, ref.alpha_exp), (out.fail, ref.fail)):
            assert torch.equal(a, r)
