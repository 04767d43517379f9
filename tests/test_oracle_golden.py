"""The CPU oracle is pinned to the live reference's outputs (tests/golden,
made by tools/make_golden.py from hessrq's numba backend)."""

import numpy as np
import pytest

from conftest import golden


def test_hypot_matches_glibc_fixture():
    import ctypes

    g = golden("scalars")
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    out = np.array([libm.hypot(a, b) for a, b in zip(g["hx"], g["hy"])])
    assert np.array_equal(out, g["hypot"])


def test_protect_update_and_pow2floor(oracle):
    g = golden("scalars")
    om = float(g["omega"])
    out = np.array([oracle.protect_update(a, b, c, om) for a, b, c in zip(g["pb"], g["ph"], g["px"])])
    assert np.array_equal(out, g["protect"])
    assert np.array_equal(np.array([oracle.pow2floor(v) for v in g["p2in"]]), g["p2out"])


def test_tile_kernels_bitwise(oracle):
    g = golden("tiles")
    for t in range(int(g["ntiles"])):
        k, b, has_left, st_r, st_s, st_cr, st_cs = (int(v) for v in g[f"t{t}_meta"])
        om = float(g[f"t{t}_omega"])
        hd, hl = g[f"t{t}_hdiag"], g[f"t{t}_hleft"]
        st, c, s = oracle.reduce_diag(hd, hl, has_left, g[f"t{t}_lam"], g[f"t{t}_rright"])
        assert st == st_r
        assert np.array_equal(c, g[f"t{t}_c"]) and np.array_equal(s, g[f"t{t}_s"])
        st, x, be = oracle.solve_rsolve(hd, hl, has_left, g[f"t{t}_lam"], g[f"t{t}_rright"], c, s,
                                        g[f"t{t}_xin"], np.zeros(b), True, om)
        assert st == st_s
        assert np.array_equal(x, g[f"t{t}_x"])
        assert np.array_equal(np.ldexp(1.0, be), g[f"t{t}_beta"])
        st, cre, cim, cs = oracle.creduce_diag(hd, hl, has_left, g[f"t{t}_clr"], g[f"t{t}_cli"],
                                               g[f"t{t}_rr2"])
        assert st == st_cr
        assert np.array_equal(cre, g[f"t{t}_cre"]) and np.array_equal(cim, g[f"t{t}_cim"])
        assert np.array_equal(cs, g[f"t{t}_cs"])
        st, x2, be = oracle.csolve_crsolve(hd, hl, has_left, g[f"t{t}_clr"], g[f"t{t}_cli"],
                                           g[f"t{t}_rr2"], cre, cim, cs, g[f"t{t}_x2in"],
                                           np.zeros(b), True, om)
        assert st == st_cs
        assert np.array_equal(x2, g[f"t{t}_x2"])
        assert np.array_equal(np.ldexp(1.0, be), g[f"t{t}_cbeta"])


def test_full_solves(oracle, same_blas):
    """dhsrq3/chsrq3 end to end: bitwise when the BLAS kernel family matches."""
    g = golden("solves")
    for tag in g["tags"]:
        b_r, b_c, robust, mode, cplx = (int(v) for v in g[f"{tag}_cfg"])
        r = oracle.solve(g[f"{tag}_h"], g[f"{tag}_lam"], g[f"{tag}_b"], b_r, b_c, robust=bool(robust),
                         mode=("solve", "eigvec")[mode])
        xr = g[f"{tag}_x"]
        if robust:
            assert np.array_equal(r.segment_scales, g[f"{tag}_seg"]), tag
            assert np.array_equal(r.alpha, g[f"{tag}_alpha"]), tag
        if same_blas:
            assert np.array_equal(r.x, xr), tag
            if robust:
                assert np.array_equal(r.norms, g[f"{tag}_norms"]), tag
        else:
            scale = np.max(np.abs(xr)) or 1.0
            assert np.max(np.abs(r.x - xr)) <= 1e-12 * scale, tag


def test_restart_stream():
    from paper_2101_05063_b200 import rng
    from paper_2101_05063_b200.inviter import _next_start

    g = golden("scalars")
    for s, row in zip(g["seeds"], g["uoc"]):
        assert np.array_equal(rng.uniform_open_closed(int(s), 64), row)
    prev = [1e-14 * np.ones(37)]
    for att, want in zip((1, 2, 3), g["starts"]):
        v = _next_start(1e-14, 37, prev, 0x5EED, att)
        prev.append(v.copy())
        assert np.array_equal(v, want)


def test_singular_shift_reported_like_reference(oracle):
    """Exactly singular shifted systems: same shift_index / local_index as
    the reference's SingularSystemError (backsolve.py:53-59)."""
    g = golden("singular")
    ncase = 0
    for t in g["tags"]:
        h, lam = g[f"{t}_h"], g[f"{t}_lam"]
        n = h.shape[0]
        b = np.ones((n, lam.size)) + (0j if int(g[f"{t}_cplx"]) else 0)
        for b_r, b_c, shift, row in g[f"{t}_hits"]:
            with pytest.raises(oracle.OracleError) as e:
                oracle.solve(h, lam, b, int(b_r), int(b_c), robust=True, mode="solve")
            assert e.value.phase == 2
            assert (e.value.shift_index, e.value.local_index) == (shift, row)
            ncase += 1
    assert ncase >= 4


def test_henry_bitwise(oracle):
    """Henry's single sweep: oracle == live reference kernels, bit for bit
    (status word included; inf/nan positions of the unguarded overflow case)."""
    g = golden("henry")
    for t in g["tags"]:
        st, x = oracle.henry_solve(g[f"{t}_h"], g[f"{t}_lam"], g[f"{t}_b"])
        assert st == int(g[f"{t}_status"]), t
        if st == 0:
            np.testing.assert_array_equal(x, g[f"{t}_x"], err_msg=str(t))


def test_compact_codes_bitwise(oracle):
    """Stewart compact encode/decode (givens.py:90-198): oracle == reference."""
    from conftest import assert_bits as eq

    g = golden("compact")
    eq(oracle.compact_encode(g["c"], g["s"]), g["t"])
    dc, ds = oracle.compact_decode(g["t"])
    eq(dc, g["dc"]), eq(ds, g["ds"])
    t1, t2 = oracle.compact_encode(g["cre"], g["cs"], g["cim"])
    eq(t1, g["packed"][0]), eq(t2, g["packed"][1])
    dre, dim, dcs = oracle.compact_decode(g["packed"][0], g["packed"][1])
    eq(dre, g["dre"]), eq(dim, g["dim"]), eq(dcs, g["dcs"])
    kc, ks = oracle.compact_decode(g["codes"])
    eq(kc, g["kc"]), eq(ks, g["ks"])


def hessenberg_checks(a, h, q, ref_h=None, ref_q=None):
    """SPEC bounds: ||Q^T Q - I|| <= 50 n eps, ||Q^T A Q - H|| <=
    100 n eps ||A||, zeros below the subdiagonal; and, where the reduction is
    forward-stable (no graded scaling), agreement with the reference's H, Q."""
    n = a.shape[0]
    eps = np.finfo(float).eps
    na = max(np.linalg.norm(a), 1.0)
    assert np.all(np.tril(h, -2) == 0.0)
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 50 * n * eps
    assert np.linalg.norm(q.T @ a @ q - h) <= 100 * n * eps * na
    if ref_h is not None:
        assert np.linalg.norm(h - ref_h) <= 100 * n * eps * na
        assert np.linalg.norm(q - ref_q) <= 100 * n * eps * np.sqrt(n)


def test_householder_hessenberg_oracle(oracle):
    """Front-end oracle vs the live reference: same reflectors (summation
    order differs from numpy's BLAS, so agreement is to rounding); the skip
    rule leaves an already-Hessenberg input bit-identical with Q = I.  The
    graded case (last) is not forward-stable: backward-error bounds only."""
    g = golden("hessenberg")
    tags = list(g["tags"])
    for t in tags:
        a = g[f"{t}_a"]
        h, q = oracle.householder_hessenberg(a)
        fwd = t != tags[-1]
        hessenberg_checks(a, h, q, g[f"{t}_h"] if fwd else None, g[f"{t}_q"] if fwd else None)
        hessenberg_checks(a, g[f"{t}_h"], g[f"{t}_q"])  # the reference meets the same bounds
    t = tags[9]  # random_unreduced: already Hessenberg
    h, q = oracle.householder_hessenberg(g[f"{t}_a"])
    assert np.array_equal(h, g[f"{t}_a"]) and np.array_equal(q, np.eye(h.shape[0]))


def test_budget_solves(oracle, same_blas):
    """dhsrq3/chsrq3 with a caller's OverflowBudget (backsolve.py:342-346,
    golden budget.npz: omega 1 / 8 / 1e3 / 2^600): bitwise like the default budget."""
    g = golden("budget")
    try:
        for tag in g["tags"]:
            b_r, b_c, mode, cplx = (int(v) for v in g[f"{tag}_cfg"])
            oracle.set_omega(float(g[f"{tag}_omega"]))
            r = oracle.solve(g[f"{tag}_h"], g[f"{tag}_lam"], g[f"{tag}_b"], b_r, b_c,
                             mode=("solve", "eigvec")[mode])
            assert np.array_equal(r.segment_scales, g[f"{tag}_seg"]), tag
            assert np.array_equal(r.alpha, g[f"{tag}_alpha"]), tag
            xr = g[f"{tag}_x"]
            if same_blas:
                assert np.array_equal(r.x, xr), tag
            else:
                assert np.max(np.abs(r.x - xr)) <= 1e-12 * (np.max(np.abs(xr)) or 1.0), tag
    finally:
        oracle.set_omega(0.0)
