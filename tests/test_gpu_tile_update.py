"""Tile-level parity of the panel kernels (hsrq_tile_update): the
reference's update_rupdate / cupdate_crupdate and reduce_offdiag /
creduce_offdiag (numba_backend.py:109-125, 198-311, 467-490, 579-736) on
single tiles -- golden outputs of the live reference (update_tiles.npz:
full, ragged and odd tile heights, shifted (super-diagonal) and far tiles,
robust and plain, right-hand sides at 1e300 so every guard fires) -- run
through the sweep's own operand code, k_scalars and k_panel.

Bar: the scale exponent delta bitwise; b and r_left to 1e-12 relative per
column (the GEMM form A [W | Zs] sums in a different order than the
reference's rotation-by-rotation recursion and OpenBLAS dgemm)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _t(a, dev, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype)


def test_tile_update_matches_reference(dev):
    import ctypes

    from paper_2101_05063_b200 import _lib

    L = _lib.load()
    g = golden("update_tiles")
    P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
    fired = 0
    for tag in g["tags"]:
        m, k, b, cplx, shifted, robust = (int(v) for v in g[f"{tag}_cfg"])
        ht, rr, xb, bio = (_t(g[f"{tag}_{n}"], dev) for n in ("ht", "rr", "xb", "bio"))
        cre, s, lre = (_t(g[f"{tag}_{n}"], dev) for n in ("cre", "s", "lre"))
        cim = _t(g[f"{tag}_cim"], dev) if cplx else None
        lim = _t(g[f"{tag}_lim"], dev) if cplx else None
        aexp = _t(g[f"{tag}_aexp"], dev, torch.int32)
        bexp = _t(g[f"{tag}_bexp"], dev, torch.int32)
        rl = torch.empty_like(rr)
        r = L.hsrq_tile_update(m, k, b, cplx, P(ht), P(rr), P(aexp), P(xb), P(lre), P(lim), shifted,
                               P(cre), P(cim), P(s), P(bexp), P(bio), P(rl), robust, 0.0,
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert r == 0, (tag, _lib.last_error())
        torch.cuda.synchronize()
        want_beta = g[f"{tag}_out_beta"]
        got_beta = np.ldexp(1.0, bexp.cpu().numpy())
        if robust:
            assert np.array_equal(got_beta, want_beta), (tag, got_beta, want_beta)
            fired += int(np.any(want_beta < np.ldexp(1.0, g[f"{tag}_bexp"])))
        for name, got in (("out_b", bio), ("out_rleft", rl)):
            want = g[f"{tag}_{name}"]
            gt = got.cpu().numpy()
            for l in range(want.shape[1]):
                sc = np.max(np.abs(want[:, l])) or 1.0
                assert np.max(np.abs(gt[:, l] - want[:, l])) <= 1e-12 * sc, (tag, name, l)
    assert fired >= 8
