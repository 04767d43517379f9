"""Every diagonal-sweep and backtransform variant the solver can select, pinned
to the oracle and to each other.

``diag_pick`` (hsrq_kernels.cu) chooses the lanes per shift DP of the
diagonal sweep from the shift count, and ``bt_launch``
(hsrq_backtransform.cuh) the backtransform lanes per shift G the same way:
config 5 on one GPU runs the warp-pair complex sweep at DP 4 with the
one-warp real sweep at DP 4 and G = 8; its 1/2, 1/4 and 1/8 shards run DP 8,
16 and 32 and G up to 32.  Small test cases select DP 32 / G 32
automatically, so here every variant is FORCED (``hsrq_tune_diag`` and
``HSRQ_BT_G``) on cases whose guards fire (start vectors at 1e300), ragged
tiles and both kinds of shifts, and each one must

* match the CPU oracle (K/numba_backend.py:75-375, 420-822 restated in
  oracle/hsrq_oracle.c) at the tolerances of test_gpu_scaling.py, and
* be bitwise identical to every other variant (X, segment / alpha exponents,
  norms, log2 norms, rotation tables, failure codes): the variants change
  only which lanes do the work, never an operation or its order.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(ROOT, "tools"))

# (DP, real DW, complex DW, real warp pairs, complex warp pairs): the one-GPU
# config-5 choice first, then the shard choices (diag_pick), then the other
# compiled warp-pair shapes
# (the 6th entry, where present: rotation-ahead pairs per CTA, hsrq_tune_diag_rx;
# 0 = off; -1 = automatic, which at a forced 32 lanes per shift stays off)
DIAG_VARIANTS = [
    (4, 4, 2, 0, 2),    # config 5, one GPU (automatic)
    (4, 4, 2, 0, 0),    # one-warp complex sweep at DP 4
    (4, 4, 2, 2, 2),    # real warp pairs too (automatic for real-only groups)
    (8, 6, 4, 0, 0),    # 1/2 shard
    (8, 6, 4, 2, 2),
    (16, 16, 16, 0, 0),  # 1/4 shard
    (16, 16, 16, 2, 2),
    (32, 16, 16, 0, 0),  # one warp per shift
    (32, 16, 16, 4, 4),
    (16, 16, 16, 0, 0, 8),  # 1/8 shard (automatic): 16-lane rotation-ahead pairs
    (16, 16, 16, 0, 0, 4),
    (32, 16, 16, 0, 0, 8),
]
BT_GS = [4, 8, 16, 32]

CASES = [  # n, b_r, seed, rhs scale, real shifts, complex shifts
    (1000, 128, 4, 1e300, 10, 14),
    (700, 64, 1, 1.0, 9, 12),
    (515, 100, 6, 1e300, 8, 9),
    (300, 37, 7, 1e300, 6, 7),
]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture
def lib(dev, monkeypatch):
    from paper_2101_05063_b200 import _lib

    L = _lib.load()
    yield L
    L.hsrq_tune_diag(0, 0, 0, -1, -1)  # back to the automatic choice
    L.hsrq_tune_diag_rx(-1)
    monkeypatch.delenv("HSRQ_BT_G", raising=False)


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


def _align(x, ref):
    ip = np.vdot(x, ref)
    return x * (ip / abs(ip)) if ip != 0 else x


def _outputs(gs):
    return {k: getattr(gs, k).cpu().numpy().copy() for k in
            ("X", "seg_exp", "alpha_exp", "norms", "log2norm", "c_re", "c_im", "s", "fail")}


def _check_oracle(h, er, ec, start, b_r, out, oracle):
    """test_gpu_scaling.py's bar: exponents exact (tile 0 / alpha +-1: the
    rounding-level final pivot of an eigenvalue shift), vectors phase-aligned
    to 1e-8, residual <= 10 n eps, represented norms within a factor 16."""
    n = h.shape[0]
    mc = ec.size
    o_c = oracle.solve(h, ec, np.repeat(start[:, None], mc, 1).astype(complex), b_r, mode="eigvec")
    o_r = oracle.solve(h, er, np.repeat(start[:, None], er.size, 1), b_r, mode="eigvec")
    seg = out["seg_exp"]
    want = np.concatenate([o_c.segment_exp, o_r.segment_exp], axis=1)
    assert np.array_equal(seg[1:], want[1:])
    assert np.max(np.abs(seg[0] - want[0])) <= 1
    assert np.max(np.abs(out["alpha_exp"] - np.concatenate([o_c.alpha_exp, o_r.alpha_exp]))) <= 1
    X = out["X"]
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
    assert np.all(np.abs(out["log2norm"] - np.concatenate([o_c.log2norm, o_r.log2norm])) < 4.0)


def _same(a, b, what):
    for k in a:
        assert np.array_equal(a[k], b[k], equal_nan=True), (what, k)


@pytest.mark.parametrize("n,b_r,seed,rhs,nr,nc", CASES)
def test_diag_variants_match_oracle_and_each_other(dev, lib, oracle, n, b_r, seed, rhs, nr, nc):
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h, er, ec = _case(n, seed, nr, nc)
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = (rho if rhs == 1.0 else rhs) * np.ones(n)
    B = torch.from_numpy(start).to(dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    base = None
    for v in DIAG_VARIANTS:
        lib.hsrq_tune_diag(*v[:5])
        lib.hsrq_tune_diag_rx(v[5] if len(v) > 5 else 0)
        gs = GroupSolver(dh, b_r, ec.size, er.size)
        gs.set_shifts(ec, er)
        assert gs.launch(B, True) == 0
        out = _outputs(gs)
        if base is None:
            if rhs > 1.0:  # the guards fired, so the variants' guard paths are compared
                assert out["seg_exp"].min() < 0
            _check_oracle(h, er, ec, start, b_r, out, oracle)
            base = out
        else:
            _same(base, out, f"diag variant {v}")


@pytest.mark.parametrize("n,b_r,seed,rhs,nr,nc", CASES[:3])
def test_backtransform_lanes_match_oracle_and_each_other(dev, lib, oracle, monkeypatch, n, b_r,
                                                         seed, rhs, nr, nc):
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h, er, ec = _case(n, seed, nr, nc)
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    start = (rho if rhs == 1.0 else rhs) * np.ones(n)
    B = torch.from_numpy(start).to(dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    lib.hsrq_tune_diag(*DIAG_VARIANTS[0])
    lib.hsrq_tune_diag_rx(0)
    base = None
    for g in BT_GS:
        monkeypatch.setenv("HSRQ_BT_G", str(g))
        gs = GroupSolver(dh, b_r, ec.size, er.size)
        gs.set_shifts(ec, er)
        assert gs.launch(B, True) == 0
        out = _outputs(gs)
        if base is None:
            _check_oracle(h, er, ec, start, b_r, out, oracle)
            base = out
        else:
            _same(base, out, f"backtransform G={g}")


def test_variants_solve_mode_explicit_rhs(dev, lib):
    """System-solve mode (dhsrq3/chsrq3, backsolve.py:316-388) with explicit
    right-hand sides: every diag / backtransform variant bitwise the same."""
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    h, er, ec = _case(640, 11, 8, 11)
    er, ec = er + 0.125, ec + 0.125j
    n = h.shape[0]
    rng = np.random.default_rng(3)
    B = torch.from_numpy(rng.standard_normal((2 * ec.size + er.size, n))).to(dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    base = None
    for v in DIAG_VARIANTS:
        for g in (8, 32):
            os.environ["HSRQ_BT_G"] = str(g)
            lib.hsrq_tune_diag(*v[:5])
            lib.hsrq_tune_diag_rx(v[5] if len(v) > 5 else 0)
            gs = GroupSolver(dh, 128, ec.size, er.size)
            gs.set_shifts(ec, er)
            assert gs.launch(B, False, mode="solve") == 0
            out = _outputs(gs)
            if base is None:
                base = out
            else:
                _same(base, out, f"solve mode {v} G={g}")
    os.environ.pop("HSRQ_BT_G", None)


def test_production_selection_at_scale_is_variant_invariant(dev, lib):
    """The automatic choice at config-5 shift counts (DP 4, warp pairs, G 8)
    against the 1/8-shard choice (DP 32, G 32) forced on the same group, at
    n = 2048 with >= 1600 shifts (the automatic pick at this count is DP 4 / G 8):
    bitwise the same."""
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    n = 2048
    h = instances.random_hessenberg(n, 21)
    rng = np.random.default_rng(21)
    ev = np.linalg.eigvals(h)
    er = ev[ev.imag == 0].real
    ec = ev[ev.imag > 0]
    # pad to config-5-like counts with perturbed copies (still near-eigenvalue shifts)
    er = np.concatenate([er, er[rng.integers(0, er.size, max(0, 700 - er.size))] * (1 + 1e-9)])
    ec = np.concatenate([ec, ec[rng.integers(0, ec.size, max(0, 900 - ec.size))] * (1 + 1e-9)])
    ec = ec[np.argsort(ec.imag, kind="stable")]
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    B = torch.full((n,), rho, dtype=torch.float64, device=dev)
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    outs = []
    for v, g in ((None, None), ((32, 16, 16, 0, 0), "32"), ((8, 6, 4, 0, 0), "16"),
                 ((16, 16, 16, 0, 0, 8), "32")):
        if v is None:
            lib.hsrq_tune_diag(0, 0, 0, -1, -1)
            lib.hsrq_tune_diag_rx(-1)
            os.environ.pop("HSRQ_BT_G", None)
        else:
            lib.hsrq_tune_diag(*v[:5])
            lib.hsrq_tune_diag_rx(v[5] if len(v) > 5 else 0)
            os.environ["HSRQ_BT_G"] = g
        gs = GroupSolver(dh, 128, ec.size, er.size)
        gs.set_shifts(ec, er)
        assert gs.launch(B, True) == 0
        outs.append(_outputs(gs))
        del gs
    os.environ.pop("HSRQ_BT_G", None)
    _same(outs[0], outs[1], "auto vs DP32/G32")
    _same(outs[0], outs[2], "auto vs DP8/G16")
    _same(outs[0], outs[3], "auto vs rotation-ahead DP16 pairs/G32")


@pytest.mark.parametrize("n,seed,rhs,nr,nc,la", [
    (1000, 4, 1e300, 10, 14, "0"), (700, 1, 1.0, 9, 12, "1"), (1300, 6, 1e300, 30, 40, "0"),
    (640, 3, 1e300, 5, 6, "1")])
def test_panel_cluster_form_is_bitwise_the_single_cta_form(dev, lib, monkeypatch, n, seed, rhs, nr,
                                                           nc, la):
    """k_panel_cl (a tile row over a 2-CTA cluster, maxima exchanged through
    distributed shared memory) vs k_panel's fast path, b_r = 128, guards
    firing (rhs 1e300), lookahead on / off, eigvec and solve modes: bitwise."""
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg, GroupSolver

    monkeypatch.setenv("HSRQ_LOOKAHEAD", la)
    h, er, ec = _case(n, seed, nr, nc)
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(h), axis=1))
    dh = DeviceHessenberg(HessenbergMatrix(h), dev)
    rng = np.random.default_rng(seed)
    cases = [(torch.full((n,), rho if rhs == 1.0 else rhs, dtype=torch.float64, device=dev), True,
              "eigvec"),
             (torch.from_numpy(rng.standard_normal((2 * ec.size + er.size, n))).to(dev), False,
              "solve")]
    try:
        for B, bc, mode in cases:
            outs = []
            for cl in (0, 1):
                lib.hsrq_tune_panel(cl)
                gs = GroupSolver(dh, 128, ec.size, er.size)
                gs.set_shifts(ec + (0.125j if mode == "solve" else 0), er + (0.125 if mode == "solve" else 0))
                assert gs.launch(B, bc, mode=mode) == 0
                outs.append(_outputs(gs))
            _same(outs[0], outs[1], f"panel cluster {mode}")
    finally:
        lib.hsrq_tune_panel(1)
