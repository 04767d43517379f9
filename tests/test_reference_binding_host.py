"""Host-side checks of the reference binding (no GPU): install / uninstall
swap the seam attribute, and the module exposes the reference's signature."""

import inspect
import types

from paper_2101_05063_b200 import reference_binding as rb


def test_install_swaps_the_seam():
    mod = types.SimpleNamespace(_solve_group=lambda *a: "cpu")
    orig = rb.install(mod)
    assert mod._solve_group is rb.solve_group_b200
    rb.uninstall(mod, orig)
    assert mod._solve_group() == "cpu"


def test_signature_matches_reference_seam():
    # inviter.py:91: _solve_group(h, grid, eigs, b, config, workspace, cplx)
    assert list(inspect.signature(rb.solve_group_b200).parameters) == [
        "h", "grid", "eigs", "b", "config", "workspace", "cplx"]
