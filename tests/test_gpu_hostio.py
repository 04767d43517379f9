"""The drop-in API's host I/O (csrc/hsrq_hostio.cuh): hsrq_h_upload and
hsrq_pack_download, and hsrq3in assembled through them.

* upload: C- and F-ordered arrays land as the same column-major device H,
  bit for bit; the device-side checks equal HessenbergMatrix's host ones
  (core.py:60-98): the infinity norm bitwise (left-to-right row sums, numpy's
  order on the reference's F-order copy), the structure check (ConfigError)
  and unreducedness -- at n > 2048, where only the device checks.
* pack: caller-order complex / real assembly with conjugation, bitwise
  against numpy.
* hsrq3in (inviter.py:186-254) through the device assembly equals the
  per-kind results of solver.solve_group put together on the host.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.mark.parametrize("n", [1, 2, 5, 257, 3001, 4096])
def test_upload_layouts_and_checks_match_hessenberg_matrix(dev, n):
    import instances
    from paper_2101_05063_b200.core import HessenbergMatrix
    from paper_2101_05063_b200.solver import DeviceHessenberg

    h = instances.random_hessenberg(n, 7) if n > 1 else np.array([[2.5]])
    h[0, -1] = -1e300 if n > 2 else h[0, -1]  # a large entry in the norm
    want = HessenbergMatrix(h)
    for arr in (np.ascontiguousarray(h), np.asfortranarray(h)):
        dh = DeviceHessenberg.upload(arr, dev)
        got = dh.t[:, :n].cpu().numpy()  # row j = column j
        assert np.array_equal(got.view(np.int64), np.ascontiguousarray(h.T).view(np.int64))
        assert dh.norm_inf == want.infinity_norm()
        assert dh.unreduced == want.is_unreduced()


def test_upload_device_structure_check(dev):
    import instances
    from paper_2101_05063_b200 import ConfigError
    from paper_2101_05063_b200.solver import DeviceHessenberg

    n = 3000
    h = instances.random_hessenberg(n, 1)
    h[2999, 2997] = 1e-300  # just below the subdiagonal
    for arr in (np.ascontiguousarray(h), np.asfortranarray(h)):
        with pytest.raises(ConfigError, match="below the first subdiagonal"):
            DeviceHessenberg.upload(arr, dev)
    h[2999, 2997] = 0.0
    h[1500, 1499] = 0.0
    dh = DeviceHessenberg.upload(h, dev)
    assert not dh.unreduced


@pytest.mark.parametrize("cplx", [True, False])
def test_pack_download_bitwise(dev, cplx):
    from paper_2101_05063_b200.inviter import _pack, _Solved
    from paper_2101_05063_b200.parallel import _NStub

    rng = np.random.default_rng(3)
    n, ncol, m = 1037, 300, 211
    X = rng.standard_normal((ncol, n))
    re = rng.integers(0, ncol - 1, m)
    im = np.where(rng.random(m) < 0.5, re + 1, -1) if cplx else np.full(m, -1)
    sg = np.where(rng.random(m) < 0.5, -1.0, 1.0)
    s = _Solved(dh=_NStub(n), X=torch.from_numpy(X).to(dev), col_r=None, col_c=None, meta=None,
                launches=0, N=0)
    got = _pack(s, re, im, sg, cplx)
    if cplx:
        imv = np.where((im >= 0)[:, None], X[np.maximum(im, 0)] * sg[:, None], 0.0)
        want = (X[re] + 1j * imv).T
    else:
        want = X[re].T
    assert got.shape == (n, m) and got.flags.c_contiguous
    assert np.array_equal(np.ascontiguousarray(want).view(np.int64), got.view(np.int64))


def test_hsrq3in_equals_solve_group_assembly(dev):
    import instances
    from paper_2101_05063_b200 import InviterConfig, hsrq3in, solver

    n = 700
    h = instances.random_hessenberg(n, 12)
    ev = np.linalg.eigvals(h)
    rng = np.random.default_rng(12)
    sel = np.concatenate([ev[ev.imag == 0][:9], ev[ev.imag > 0][:10], ev[ev.imag < 0][10:16]])
    sel = sel[rng.permutation(sel.size)]
    res = hsrq3in(np.ascontiguousarray(h), sel, InviterConfig(b_r=128, max_restarts=0))
    is_c = sel.imag != 0
    er = sel[~is_c].real
    ec = np.where(sel[is_c].imag < 0, sel[is_c].conj(), sel[is_c])
    rho = np.finfo(float).eps * np.max(np.sum(np.abs(np.asfortranarray(h)), axis=1))
    out, _ = solver.solve_group(h, ec, er, rho * np.ones(n), 128)
    X = out.X.cpu().numpy()
    mc = ec.size
    want = np.zeros((n, sel.size), dtype=complex)
    want[:, ~is_c] = X[2 * mc:].T
    xc = (X[0:2 * mc:2] + 1j * X[1:2 * mc:2]).T
    flip = sel[is_c].imag < 0
    xc[:, flip] = xc[:, flip].conj()
    want[:, is_c] = xc
    assert np.array_equal(res.vectors.view(np.int64), want.view(np.int64))
    assert res.converged.all()
    seg = out.seg_exp.cpu().numpy()
    ws = np.zeros_like(res.segment_exp)
    ws[:, ~is_c] = seg[:, mc:]
    ws[:, is_c] = seg[:, :mc]
    assert np.array_equal(res.segment_exp, ws)
