"""INTEGRATION.md's raw-ctypes stub (`henry_solve_b200`, the binding a
maintainer of the reference would add for the single-sweep baseline) is
executed verbatim from the document against the live reference's kernel
outputs (golden henry.npz): the published recipe itself is under test, not
a copy of it."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _stub_namespace():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        doc = f.read()
    blocks = re.findall(r"```python\n(.*?)```", doc, flags=re.S)
    code = next(b for b in blocks if "def henry_solve_b200" in b)
    so = os.path.join(ROOT, "paper_2101_05063_b200", "libhsrq_b200.so")
    assert '"/path/to/paper_2101_05063_b200/libhsrq_b200.so"' in code
    code = code.replace('"/path/to/paper_2101_05063_b200/libhsrq_b200.so"', repr(so))
    ns = {}
    exec(compile(code, "INTEGRATION.md:henry_solve_b200", "exec"), ns)
    return ns


def test_integration_md_henry_stub_matches_reference_kernels():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()  # (a CUDA context for the stub's raw cudart calls)
    ns = _stub_namespace()
    g = golden("henry")
    ran = 0
    for t in g["tags"]:
        h, lam, b = g[f"{t}_h"], g[f"{t}_lam"], g[f"{t}_b"]
        if lam.ndim == 0 or b.ndim != 2:
            continue  # the stub takes the kernels' array contract: lam (m,), x (n, m)
        cplx = np.iscomplexobj(lam)
        x = np.array(b, dtype=np.complex128 if cplx else np.float64, order="C")
        st = ns["henry_solve_b200"](np.asarray(h, dtype=np.float64), np.ascontiguousarray(lam), x)
        assert st == int(g[f"{t}_status"]), t
        if st == 0:
            np.testing.assert_array_equal(x, g[f"{t}_x"].reshape(x.shape), err_msg=str(t))
        ran += 1
    assert ran >= 10


@pytest.mark.parametrize("stub", ["solve_group_b200_host", "solve_group_b200"])
def test_integration_md_solve_group_stubs_drive_the_reference(stub):
    """The two `_solve_group` stubs of INTEGRATION.md (raw ctypes + cudart with
    numpy in / out; torch device buffers) are executed verbatim as modules of
    the installed reference package and take over `hessrq.inviter._solve_group`:
    the reference's own hsrq3in must then reproduce its CPU run on H1 (golden
    inviter.npz), and an exactly singular shift must raise with the
    reference's indices."""
    import sys
    import types

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hessrq")):
        pytest.skip("hessrq not installed under baseline/_ref")
    sys.path.insert(0, ref)
    import hessrq.inviter as inv

    torch.cuda.init()
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        doc = f.read()
    code = next(b for b in re.findall(r"```python\n(.*?)```", doc, flags=re.S)
                if f"def {stub}(" in b)
    so = os.path.join(ROOT, "paper_2101_05063_b200", "libhsrq_b200.so")
    code = code.replace('"/path/to/paper_2101_05063_b200/libhsrq_b200.so"', repr(so))
    mod = types.ModuleType(f"hessrq._b200_stub_{stub}")
    mod.__package__ = "hessrq"  # the stub's `from .core import ...`
    exec(compile(code, f"INTEGRATION.md:{stub}", "exec"), mod.__dict__)
    orig = inv._solve_group
    inv._solve_group = getattr(mod, stub)
    try:
        g = golden("inviter")
        h, eigs = g["h1_h"], g["h1_eigs"]
        r = inv.hsrq3in(h, eigs, inv.InviterConfig(b_r=8, b_c=4))
        assert np.array_equal(r.converged, g["h1_conv"])
        assert np.array_equal(r.restarts, g["h1_restarts"])
        want = g["h1_vectors"] if "h1_vectors" in g.files else None
        hf = np.linalg.norm(h, "fro")
        for l in range(eigs.size):
            x = r.vectors[:, l]
            if want is not None:
                w = want[:, l]
                ip = np.vdot(x, w)
                assert np.linalg.norm(x * (ip / abs(ip)) - w) <= 1e-8
            res = np.linalg.norm(h @ x - eigs[l] * x) / (hf * np.linalg.norm(x))
            assert res <= 10 * h.shape[0] * np.finfo(float).eps
        from paper_2101_05063_b200 import SingularSystemError

        s = golden("singular")
        t = s["tags"][0]
        hs, lam = s[f"{t}_h"], s[f"{t}_lam"]
        try:  # one tile (b_r = n): the zero pivot is reproduced exactly
            inv.hsrq3in(hs, np.array([lam[1]]), inv.InviterConfig(b_r=hs.shape[0], b_c=2))
        except SingularSystemError as e:
            assert (e.shift_index, e.local_index) == (0, 0)
        else:
            raise AssertionError("the exactly singular shift did not raise")
    finally:
        inv._solve_group = orig
