"""Edge inputs of the inverse-iteration drivers on the GPU path against what
the live reference returned or raised for them (golden edge.npz, made by
tools/make_golden.py gen_edge): n = 1, 2, 3, a one-row ragged last tile, a
single shift of either kind, only Im < 0 shifts, repeated shifts, a mixed
caller order, empty selections, the wrong driver for the shift kind."""

import warnings

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cases():
    g = golden("edge")
    return [str(t) for t in g["tags"]]


@pytest.mark.parametrize("tag", _cases())
def test_edge_input_behaves_like_reference(tag):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_05063_b200 as P

    g = golden("edge")
    h, eigs, b_r = g[f"{tag}_h"], g[f"{tag}_eigs"], int(g[f"{tag}_br"])
    fn = getattr(P, str(g[f"{tag}_fn"]))
    want_err = str(g[f"{tag}_error"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # the reference's own ComplexWarning on a real-driver cast
        if want_err:
            with pytest.raises(Exception) as e:
                fn(h, eigs, P.InviterConfig(b_r=b_r))
            assert type(e.value).__name__ in (want_err, {"TaskError": "SingularTaskError"}.get(want_err))
            assert isinstance(e.value, getattr(P, want_err))
            assert str(e.value) == str(g[f"{tag}_message"])
            return
        r = fn(h, eigs, P.InviterConfig(b_r=b_r))
    want = g[f"{tag}_vectors"]
    assert r.vectors.shape == want.shape
    assert np.array_equal(r.converged, g[f"{tag}_conv"])
    assert np.array_equal(r.restarts, g[f"{tag}_restarts"])
    n = h.shape[0]
    hf = np.linalg.norm(h, "fro")
    lam = np.asarray(eigs)
    if str(g[f"{tag}_fn"]) == "dhsrq3in":
        lam = lam.real
    for l in range(want.shape[1]):
        x, w = np.asarray(r.vectors[:, l], dtype=complex), want[:, l]
        if not g[f"{tag}_conv"][l]:
            assert not np.any(x) and not np.any(w)  # zero-filled, flagged
            continue
        ip = np.vdot(x, w)  # phase-aligned (north_star): the phase is pivot-rounding noise
        assert abs(abs(ip) - 1.0) <= 1e-8
        assert np.linalg.norm(x * (ip / abs(ip)) - w) <= 1e-8
        res = np.linalg.norm(h @ x - lam[l] * x) / (hf * np.linalg.norm(x))
        assert res <= 10 * n * np.finfo(float).eps
