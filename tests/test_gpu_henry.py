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
