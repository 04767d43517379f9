"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/hsrq.h declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "hsrq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hsrq_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("hsrq_solve_group", "hsrq_solve_group_async", "hsrq_workspace_bytes",
                 "hsrq_tile_diag", "hsrq_protect_update_batch", "hsrq_hypot_batch"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2101_05063_b200 import _lib

    lib = _lib.load()
    raw = ctypes.CDLL(lib._name)
    for name in _declared():
        assert hasattr(raw, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_host_only_entry_points():
    from paper_2101_05063_b200 import _lib

    lib = _lib.load()
    assert lib.hsrq_version().decode().startswith("hsrq_b200")
    ws = lib.hsrq_workspace_bytes(16000, 128, 6105, 3790)
    # crossover store n x cols plus the B operand: O(n * cols), not O(n * N * cols)
    assert 16000 * 16000 * 8 < ws < 3 * 16000 * 16000 * 8
    assert lib.hsrq_workspace_bytes(0, 128, 1, 1) == 0


def test_sass_is_sm100a_with_dmma():
    """The shipped kernels are sm_100a code and the panel GEMM issues DMMA."""
    import shutil
    import subprocess

    from paper_2101_05063_b200 import _build

    if not shutil.which("cuobjdump"):
        return
    out = subprocess.run(["cuobjdump", "-sass", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out
