"""The reference package's OWN inverse-iteration drivers with its seam swapped
for the B200 library (paper_2101_05063_b200.reference_binding, the binding
INTEGRATION.md describes).

``hessrq`` is imported from ``baseline/_ref`` (an unmodified
``pip install --no-deps --target baseline/_ref`` of /root/reference, made in
the build container; it travels to the GPU box with the repo snapshot).
Where it is absent the tests skip.  With ``hessrq.inviter._solve_group``
routed to ``solve_group_b200``, the reference's ``hsrq3in`` / ``dhsrq3in`` /
``chsrq3in`` / ``_iterate`` (inviter.py:109-254: restarts, convergence,
grouping, ordering -- all reference code) must reproduce the golden outputs
of the reference's CPU run, and exactly singular shifts must raise what the
reference raises: its own TaskError around its SingularSystemError.
"""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def inviter():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "hessrq")):
        pytest.skip("hessrq not installed under baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import hessrq.inviter as inv
    except Exception as e:  # pragma: no cover
        pytest.skip(f"hessrq not importable: {e}")
    from paper_2101_05063_b200 import reference_binding

    assert inv.__file__.startswith(REF)
    orig = reference_binding.install(inv)
    yield inv
    reference_binding.uninstall(inv, orig)


def _align(x, ref):
    ip = np.vdot(x, ref)
    return x * (ip / abs(ip)) if ip != 0 else x


def test_reference_drivers_on_the_b200_seam_h1(inviter):
    g = golden("inviter")
    h, eigs = g["h1_h"], g["h1_eigs"]
    cfg = inviter.InviterConfig(b_r=8, b_c=4)
    r = inviter.hsrq3in(h, eigs, cfg)
    assert np.array_equal(r.converged, g["h1_conv"])
    assert np.array_equal(r.restarts, g["h1_restarts"])
    for l in range(eigs.size):
        want = g["h1_vectors"][:, l]
        assert np.linalg.norm(_align(r.vectors[:, l], want) - want) <= 1e-8
    sel = eigs[eigs.imag > 0]
    rc = inviter.chsrq3in(h, sel.conj(), cfg)
    for l in range(sel.size):
        want = g["h1c_vectors"][:, l]
        assert np.linalg.norm(_align(rc.vectors[:, l], want) - want) <= 1e-8
    rr = inviter.dhsrq3in(h, eigs[eigs.imag == 0].real, cfg)
    assert np.array_equal(rr.restarts, g["h1r_restarts"])
    for l in range(rr.vectors.shape[1]):
        want = g["h1r_vectors"][:, l]
        assert np.linalg.norm(_align(rr.vectors[:, l], want) - want) <= 1e-8


def test_reference_restarts_on_the_b200_seam(inviter):
    g = golden("inviter")
    r = inviter.dhsrq3in(g["rs_h"], g["rs_shifts"], inviter.InviterConfig(b_r=5, b_c=2))
    assert np.array_equal(r.converged, g["rs_conv"])
    assert np.array_equal(r.restarts, g["rs_restarts"])
    assert r.restarts.max() > 0
    for l in np.nonzero(r.converged)[0]:
        want = g["rs_vectors"][:, l]
        assert np.linalg.norm(_align(r.vectors[:, l], want) - want) <= 1e-8


def test_reference_config1_on_the_b200_seam(inviter):
    g = golden("inviter")
    h, shifts = g["c1_h"], g["c1_shifts"]
    r = inviter.hsrq3in(h, shifts, inviter.InviterConfig(b_r=32))
    assert np.array_equal(r.converged, g["c1_conv"])
    assert np.array_equal(r.restarts, g["c1_restarts"])
    n = h.shape[0]
    hf = np.linalg.norm(h, "fro")
    for l in range(shifts.size):
        x = r.vectors[:, l]
        want = g["c1_vectors"][:, l]
        assert np.linalg.norm(_align(x, want) - want) <= 1e-8
        assert np.linalg.norm(h @ x - shifts[l] * x) / (hf * np.linalg.norm(x)) <= 10 * n * np.finfo(float).eps
    # the reference's own workspace accounting saw the cross-over size of the call
    assert r.peak_crossover_reals == n * (n // 32) * shifts.size


def test_reference_singular_shift_raises_reference_error(inviter):
    """hsrq3in on an exactly singular shift: what the reference's caller sees --
    the reference's own TaskError (scheduler.py:182-187) with the node, message
    and SingularSystemError cause of the reference's CPU run (or, across
    tiles, a converged vector: test_gpu_configs.py documents why)."""
    import hessrq.core as rcore
    import hessrq.scheduler as rsched

    g = golden("singular")
    kinds = [str(k) for k in g["node_kinds"]]
    seen = 0
    for t in g["tags"]:
        h, lam = g[f"{t}_h"], g[f"{t}_lam"]
        want = tuple(g[f"{t}_inviter"])
        node = g[f"{t}_inviter_node"]
        try:
            r = inviter.hsrq3in(h, np.array([lam[1]]), inviter.InviterConfig(b_r=3, b_c=2))
        except rsched.TaskError as e:
            assert type(e) is rsched.TaskError and isinstance(e.cause, rcore.SingularSystemError)
            assert e.__cause__ is e.cause
            assert (e.cause.shift_index, e.cause.local_index) == want
            assert isinstance(e.node, rsched.TaskNode) and e.node.kind == kinds[node[0]]
            assert tuple(e.node.coords) == tuple(int(v) for v in node[1:4])
            assert e.node.seq == node[4]
            assert str(e) == str(g[f"{t}_inviter_message"])
            seen += 1
        else:
            assert r.converged[0]
    print(f"{seen} of {len(g['tags'])} singular shifts raised (the rest converged across tiles)")
