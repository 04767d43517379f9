"""Stewart compact rotation storage on the GPU (givens.py:90-198,
GivensTable.compact / from_compact core.py:193-209): device codes bitwise
equal to the reference's, and solves that store their rotations compactly
(HSRQ_MODE_COMPACT_ROTATIONS) agree with the full-table solves."""

import numpy as np
import pytest

from conftest import assert_bits, golden

pytestmark = pytest.mark.gpu


def test_device_codes_match_reference():
    import torch

    from paper_2101_05063_b200.solver import compact_decode, compact_encode

    g = golden("compact")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    C = lambda t: t.cpu().numpy()
    assert_bits(C(compact_encode(T(g["c"]), None, T(g["s"]))), g["t"])
    dc, ds = compact_decode(T(g["t"]))
    assert_bits(C(dc), g["dc"]), assert_bits(C(ds), g["ds"])
    t1, t2 = compact_encode(T(g["cre"]), T(g["cim"]), T(g["cs"]))
    assert_bits(C(t1), g["packed"][0]), assert_bits(C(t2), g["packed"][1])
    dre, dim, dcs = compact_decode(T(g["packed"][0]), T(g["packed"][1]))
    assert_bits(C(dre), g["dre"]), assert_bits(C(dim), g["dim"]), assert_bits(C(dcs), g["dcs"])
    kc, ks = compact_decode(T(g["codes"]))
    assert_bits(C(kc), g["kc"]), assert_bits(C(ks), g["ks"])


@pytest.mark.parametrize("mode", ["eigvec", "solve"])
def test_compact_solve_matches_full_tables(mode):
    """Mixed real/complex group, ragged last tile: the compact table is the
    encoding of the full table bit for bit; scales and norms are identical;
    vectors agree to rounding (decoded rotations differ from the exact ones
    in the last bits)."""
    import torch

    from paper_2101_05063_b200.solver import compact_encode, solve_group

    rng = np.random.default_rng(11)
    n, b_r = 700, 64
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    er = rng.uniform(-3, 3, 9)
    ec = rng.uniform(-3, 3, 7) + 1j * rng.uniform(0.1, 2, 7)
    b = rng.standard_normal(n)
    full, _ = solve_group(h, ec, er, b, b_r, mode=mode)
    Xf = full.X.cpu().numpy().copy()
    cr, ci, s = (t.clone() for t in full.rotations())
    segf, nf = full.seg_exp.cpu().numpy().copy(), full.norms.cpu().numpy().copy()
    comp, _ = solve_group(h, ec, er, b, b_r, mode=mode, compact=True)
    assert comp.nfail == 0 and full.nfail == 0
    mc = ec.size
    t1, t2 = compact_encode(cr[:mc], ci[:mc], s[:mc])
    assert_bits(comp.c_re[:mc].cpu().numpy(), t1.cpu().numpy())
    assert_bits(comp.c_im[:mc].cpu().numpy(), t2.cpu().numpy())
    assert_bits(comp.c_re[mc:].cpu().numpy(), compact_encode(cr[mc:], None, s[mc:]).cpu().numpy())
    assert np.array_equal(comp.seg_exp.cpu().numpy(), segf)
    assert_bits(comp.norms.cpu().numpy(), nf)
    Xc = comp.X.cpu().numpy()
    rel = np.max(np.abs(Xc - Xf), axis=1) / np.max(np.abs(Xf), axis=1)
    assert rel.max() < 1e-12, rel.max()
    dre, dim, dcs = comp.rotations()
    assert np.max(np.abs(dre.cpu().numpy() - cr.cpu().numpy())) < 1e-15 * 4


def test_inverse_iteration_with_compact_rotations():
    from paper_2101_05063_b200 import InviterConfig, hsrq3in

    rng = np.random.default_rng(2)
    n = 300
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    ev = np.linalg.eigvals(h)
    sel = np.concatenate([ev[ev.imag == 0][:5], ev[ev.imag > 0][:5], ev[ev.imag < 0][:3]])
    a = hsrq3in(h, sel, InviterConfig(b_r=64))
    c = hsrq3in(h, sel, InviterConfig(b_r=64, compact_rotations=True))
    assert np.array_equal(a.converged, c.converged)
    for l in range(sel.size):
        x, y = a.vectors[:, l], c.vectors[:, l]
        ip = np.vdot(y, x)
        assert np.linalg.norm(y * (ip / abs(ip)) - x) < 1e-10
