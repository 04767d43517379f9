"""Henry's single-sweep baseline on the GPU (k_henry_real / k_henry_cplx via
hsrq_henry_solve) against the live reference's kernels (tests/golden/henry.npz)
and the oracle: bit for bit, exceptions with the reference's indices."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _unpack(st):
    return st >> 42, (st >> 21) & ((1 << 21) - 1), st & ((1 << 21) - 1)


def test_henry_golden_bitwise():
    from paper_2101_05063_b200 import SingularSystemError, StructuralViolationError, henry_rq_solve

    g = golden("henry")
    for t in g["tags"]:
        h, lam, b = g[f"{t}_h"], g[f"{t}_lam"], g[f"{t}_b"]
        lam_in = lam.item() if lam.ndim == 0 else lam
        st = int(g[f"{t}_status"])
        if st == 0:
            x = henry_rq_solve(h, lam_in, b)
            want = g[f"{t}_x"]
            np.testing.assert_array_equal(np.asarray(x).reshape(want.shape), want, err_msg=str(t))
        else:
            kind, l, row = _unpack(st)
            exc = StructuralViolationError if kind == 1 else SingularSystemError
            with pytest.raises(exc) as ei:
                henry_rq_solve(h, lam_in, b)
            if kind == 2:
                assert (ei.value.shift_index, ei.value.local_index) == (l, row), t


@pytest.mark.parametrize("cplx", [False, True])
def test_henry_matches_oracle_larger(cplx, oracle):
    """n = 700, 37 shifts (more shifts than one wave of CTAs on small grids)."""
    from paper_2101_05063_b200 import henry_rq_solve

    rng = np.random.default_rng(5)
    n, m = 700, 37
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    lam = rng.uniform(-3, 3, m) + (1j * rng.uniform(0.1, 2, m) if cplx else 0)
    b = rng.standard_normal((n, m)) + (1j * rng.standard_normal((n, m)) if cplx else 0)
    st, want = oracle.henry_solve(h, lam, b)
    assert st == 0
    x = henry_rq_solve(h, lam, b)
    np.testing.assert_array_equal(x, want)


def test_bench_csv_rows(tmp_path):
    """python -m paper_2101_05063_b200.benchcsv writes the hessrq-bench-v1 CSV:
    one row per robust mode, per-task seconds, flop counters, henry_s."""
    import csv

    from paper_2101_05063_b200 import benchcsv

    out = tmp_path / "b.csv"
    assert benchcsv.main(["--matrix", "random:n=300,seed=1", "--shift-count", "12", "--kind",
                          "complex", "--tile-rows", "64", "--robust", "both", "--compare-henry",
                          "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert [r["robust"] for r in rows] == ["on", "off"]
    for r in rows:
        assert r["schema"] == "hessrq-bench-v1" and r["backend"] == "b200"
        assert float(r["total_s"]) > 0 and float(r["henry_s"]) > 0
        assert float(r["gpu_panel_s"]) > 0 and float(r["flops_Update"]) > 0


def test_henry_config3_sample_bitwise(oracle):
    """Config-3-sized sweep (n = 4000, random Hessenberg as in the BASELINE
    complex-shift config) on a sample of eigenvalue shifts: GPU == oracle bit
    for bit, real and complex (inf / NaN positions included).  Where the
    unguarded single sweep stays finite the result is an eigenvector
    direction; where it overflows -- the failure the paper's scaling exists
    for -- the robust tiled solve of the same shift is finite."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tools"))
    import instances
    from paper_2101_05063_b200 import chsrq3, dhsrq3, henry_rq_solve

    h = instances.make_h(3)
    ev = np.load(instances.eig_path(3))
    n = h.shape[0]
    for lam in (ev[ev.imag == 0].real[:4], ev[ev.imag > 0][:4]):
        b = np.ones((n, lam.size)) + (0j if np.iscomplexobj(lam) else 0)
        st, want = oracle.henry_solve(h, lam, b)
        assert st == 0
        x = henry_rq_solve(h, lam, b)
        np.testing.assert_array_equal(x, want)
        hf = np.linalg.norm(h, "fro")
        robust = (chsrq3 if np.iscomplexobj(lam) else dhsrq3)(h, lam, b, mode="eigvec")
        for l in range(lam.size):
            if np.all(np.isfinite(x[:, l])):
                xl = x[:, l] / np.linalg.norm(x[:, l])
            else:
                xl = robust.x[:, l]
                assert np.all(np.isfinite(xl))
            assert np.linalg.norm(h @ xl - lam[l] * xl) / hf <= 10 * n * np.finfo(float).eps


def test_dhsrq3_fills_runstats():
    """dhsrq3 / chsrq3 ``stats``: the reference's RunStats fields, exact flop
    and formula counters (= the reference's, tests/golden/runstats.npz via
    flops.task_flops), measured per-task seconds."""
    from paper_2101_05063_b200 import RunStats, chsrq3, dhsrq3, flops

    rng = np.random.default_rng(3)
    n = 300
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    for cplx in (False, True):
        lam = rng.uniform(2, 3, 5) + (0.5j if cplx else 0)
        b = np.ones((n, 5)) + (0j if cplx else 0)
        st = RunStats()
        (chsrq3 if cplx else dhsrq3)(h, lam, b, b_r=64, stats=st)
        ex, fo = flops.task_flops(n, 64, 5, cplx)
        assert st.flops == ex and st.formula == fo
        assert all(st.seconds[t] > 0 for t in flops.TASK_TYPES)
