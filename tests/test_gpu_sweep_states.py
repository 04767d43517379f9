"""Column-by-column parity of the fused sweep: the GPU state after tile
column s's panel (HSRQ_STOP_AT=s: solved tiles >= s, right-hand sides of
the tiles above updated by every column >= s, the segment exponents) against
the oracle's substitution state after the same column (oracle.set_stop).
Pins the panel GEMM and its guard logic (update_rupdate steps 1-3,
numba_backend.py:198-311 / cupdate_crupdate :579-736) tile column by tile
column, not only through the finished solve."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,n,b_r,scale", [(1, 500, 64, 1.0), (2, 620, 128, 1e300),
                                               (3, 333, 32, 1e290)])
def test_state_after_each_column(oracle, monkeypatch, seed, n, b_r, scale):
    from paper_2101_05063_b200.solver import solve_group

    rng = np.random.default_rng(seed)
    h = np.triu(rng.standard_normal((n, n)))
    h[np.arange(1, n), np.arange(n - 1)] = np.abs(rng.standard_normal(n - 1)) + 0.1
    ev = np.linalg.eigvals(h)
    er = ev[ev.imag == 0].real[:3]
    ec = ev[ev.imag > 0][:3]
    N = (n + b_r - 1) // b_r
    b = np.full(n, scale)
    try:
        for stop in sorted({N - 1, N // 2, 1}):
            monkeypatch.setenv("HSRQ_STOP_AT", str(stop))
            out, _ = solve_group(h, ec, er, b, b_r, mode="solve")
            X = out.X.cpu().numpy()
            seg = out.seg_exp.cpu().numpy()
            oracle.set_stop(stop)
            o_r = oracle.solve(h, er, np.repeat(b[:, None], er.size, 1), b_r, mode="solve")
            o_c = oracle.solve(h, ec, np.repeat(b[:, None], ec.size, 1).astype(complex), b_r,
                               mode="solve")
            mc = ec.size
            assert np.array_equal(seg, np.concatenate([o_c.segment_exp, o_r.segment_exp], 1)), stop
            got = np.concatenate([(X[0:2 * mc:2] + 1j * X[1:2 * mc:2]).T, X[2 * mc:].T], 1)
            want = np.concatenate([o_c.x, o_r.x], 1)
            err = np.max(np.abs(got - want), axis=0) / np.max(np.abs(want), axis=0)
            assert err.max() < 1e-10, (stop, err.max())
    finally:
        oracle.set_stop(-1)
