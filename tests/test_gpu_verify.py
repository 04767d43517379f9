"""The reference's own property suite (hessrq verify, verifysuite.py) run on
the GPU path: every check passes, and the corrupt-rotation hook is caught."""

import pytest

pytestmark = pytest.mark.gpu


def test_verify_suite_passes():
    from gpu_verifysuite import run_verify

    ok, rep = run_verify()
    assert ok, [c for c in rep["checks"] if not c["passed"]]
    assert len(rep["checks"]) == 8


def test_verify_suite_catches_corrupted_rotation():
    from gpu_verifysuite import run_verify

    ok, rep = run_verify(quick=True, corrupt_givens=True)
    assert not ok
    bad = [c["name"] for c in rep["checks"] if not c["passed"]]
    assert bad == ["rq_identity_real"]
