"""Out-of-bounds write check of the solve entry point (memcheck substitute:
compute-sanitizer is closed on the GPU pool).

Every output of ``hsrq_solve_group`` (include/hsrq.h) is placed inside a
larger allocation filled with a canary bit pattern, with leading dimensions
larger than n (ldx, ldc, ldh padded), and the workspace is followed by a
canary tail.  After solves that take every kernel variant and guard path
(start vectors at 1e300, ragged tiles, lookahead on and off, compact
rotations), the canaries -- guard zones before and after each buffer and
the gap rows between leading dimension and n -- must be untouched, and H must
be unchanged (the reference never writes H, core.py:60-79)."""

import ctypes
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
sys.path.insert(0, os.path.join(ROOT, "tools"))

CANARY = np.frombuffer(np.array([0x7FF4DEADBEEF1234], dtype=np.int64).tobytes(), dtype=np.float64)[0]
GUARD = 4096  # elements of canary before and after every buffer


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


class Guarded:
    """A (rows, ld) row-major device buffer (row r = column r of a column-major
    block, leading dimension ld) inside a canary-filled allocation."""

    def __init__(self, rows, ld, dtype, dev):
        esz = torch.empty(0, dtype=dtype).element_size()
        nbytes = (2 * GUARD * 8) + rows * ld * esz
        self.raw = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=dev)
        self.raw.fill_(CANARY)
        self.byte0 = GUARD * 8
        self.rows, self.ld, self.dtype, self.esz = rows, ld, dtype, esz
        self.view = self.raw.view(torch.uint8)[self.byte0:self.byte0 + rows * ld * esz].view(dtype) \
            .view(rows, ld)

    def ptr(self):
        return ctypes.c_void_p(self.raw.data_ptr() + self.byte0)

    def check(self, used_cols, what):
        raw = self.raw.view(torch.uint8).cpu().numpy()
        end = self.byte0 + self.rows * self.ld * self.esz
        assert np.array_equal(raw[: self.byte0], _pattern(0, self.byte0)), f"{what}: write before buffer"
        assert np.array_equal(raw[end:], _pattern(end, raw.size - end)), f"{what}: write past buffer"
        if used_cols < self.ld:
            for r in range(self.rows):
                a = self.byte0 + (r * self.ld + used_cols) * self.esz
                b = self.byte0 + (r + 1) * self.ld * self.esz
                assert np.array_equal(raw[a:b], _pattern(a, b - a)), \
                    f"{what}: write into the leading-dimension gap of row {r}"


def _pattern(start, size):
    """The canary bytes found at absolute byte offsets [start, start + size)."""
    cb = np.frombuffer(np.float64(CANARY).tobytes(), dtype=np.uint8)
    return np.resize(np.roll(cb, -(start % 8)), size)


@pytest.mark.parametrize("n,b_r,seed,la,compact,dp", [
    (300, 64, 3, "1", False, (4, 4, 2, 0, 2)),
    (300, 64, 3, "0", True, (32, 16, 16, 4, 4)),
    (515, 100, 6, "1", False, (8, 6, 4, 2, 2)),
    (515, 128, 6, "0", False, (16, 16, 16, 0, 0)),
    (130, 128, 2, "1", True, (0, 0, 0, -1, -1)),
])
def test_no_out_of_bounds_writes(dev, monkeypatch, n, b_r, seed, la, compact, dp):
    import instances
    from paper_2101_05063_b200 import _lib

    L = _lib.load()
    monkeypatch.setenv("HSRQ_LOOKAHEAD", la)
    L.hsrq_tune_diag(*dp)
    try:
        h = instances.random_hessenberg(n, seed)
        ev = np.linalg.eigvals(h)
        er = ev[ev.imag == 0].real[:9]
        ec = ev[ev.imag > 0][:13]
        mc, mr = ec.size, er.size
        ms, ncol = mc + mr, 2 * mc + mr
        N = (n + b_r - 1) // b_r
        ldh, ldx, ldc = n + 6, n, n + 3  # ldx == n: X and the crossover share a layout
        f64, i32, i64 = torch.float64, torch.int32, torch.int64
        H = Guarded(n, ldh, f64, dev)
        H.view[:, :n] = torch.from_numpy(np.ascontiguousarray(h.T)).to(dev)  # row j = column j
        h_before = H.raw.clone()
        lam = np.concatenate([ec, er.astype(complex)])
        lre = Guarded(1, ms, f64, dev)
        lim = Guarded(1, ms, f64, dev)
        lre.view[0] = torch.from_numpy(lam.real.copy()).to(dev)
        lim.view[0] = torch.from_numpy(lam.imag.copy()).to(dev)
        B = Guarded(1, n, f64, dev)
        B.view[0] = 1e300
        X = Guarded(ncol, ldx, f64, dev)
        cre = Guarded(ms, ldc, f64, dev)
        cim = Guarded(ms if not compact else max(mc, 1), ldc, f64, dev)
        s = Guarded(ms, ldc, f64, dev)
        seg = Guarded(N, ms, i32, dev)
        aexp = Guarded(1, ms, i32, dev)
        norms = Guarded(1, ms, f64, dev)
        l2 = Guarded(1, ms, f64, dev)
        fail = Guarded(1, ms, i64, dev)
        wsb = int(L.hsrq_workspace_bytes(n, b_r, mc, mr))
        ws = Guarded(1, (wsb + 7) // 8, f64, dev)
        st = torch.cuda.current_stream(dev)
        mode = 1 | (0x10 if compact else 0)
        r = L.hsrq_solve_group(H.ptr(), ldh, n, b_r, lre.ptr(), lim.ptr(), mc, mr, B.ptr(), 0, 1,
                               X.ptr(), ldx, cre.ptr(), cim.ptr(), s.ptr() if not compact else None,
                               ldc, seg.ptr(), aexp.ptr(), norms.ptr(), l2.ptr(), fail.ptr(), 1,
                               mode, ws.ptr(), wsb, ctypes.c_void_p(st.cuda_stream))
        assert r == 0, (r, _lib.last_error())
        torch.cuda.synchronize()
        assert torch.equal(H.raw.view(torch.int64), h_before.view(torch.int64)), "H was written"
        for buf, used, what in ((X, n, "X"), (cre, n, "c_re"), (cim, n, "c_im"), (s, n, "s"),
                                (seg, ms, "seg_exp"), (aexp, ms, "alpha_exp"),
                                (norms, ms, "norms"), (l2, ms, "log2norm"), (fail, ms, "fail"),
                                (lre, ms, "lam_re"), (lim, ms, "lam_im"), (B, n, "B")):
            buf.check(used, what)
        # the workspace's own tail (past ws_bytes)
        raw = ws.raw.view(torch.uint8).cpu().numpy()
        P = ws.byte0 + wsb
        assert np.array_equal(raw[P:], _pattern(P, raw.size - P)), "write past the workspace"
        assert np.all(np.isfinite(X.view[:, :n].cpu().numpy()))
    finally:
        L.hsrq_tune_diag(0, 0, 0, -1, -1)
