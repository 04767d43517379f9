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
