"""ctypes binding of libhsrq_b200.so (the C ABI in include/hsrq.h).

There is no CPU fallback: if the library is missing or cannot be loaded the
import of the solver fails loudly.
"""

from __future__ import annotations

import ctypes
import os

from ._build import LIB, build, stale, variant_lib

_c = ctypes
_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double
_sz = ctypes.c_size_t

# symbol -> (restype, argtypes); mirrors include/hsrq.h
SIGNATURES = {
    "hsrq_version": (ctypes.c_char_p, []),
    "hsrq_last_error": (ctypes.c_char_p, []),
    "hsrq_workspace_bytes": (_sz, [_i64, _i32, _i64, _i64]),
    "hsrq_solve_group": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _i64,
         _p, _p, _p, _p, _p, _i32, _i32, _p, _sz, _p],
    ),
    "hsrq_solve_group_omega": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _i64,
         _p, _p, _p, _p, _p, _i32, _i32, _f64, _p, _sz, _p],
    ),
    "hsrq_solve_group_async": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _i64,
         _p, _p, _p, _p, _p, _i32, _i32, _p, _sz, _p],
    ),
    "hsrq_failure_count": (_i64, [_p, _p]),
    "hsrq_graph_capture": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _i64,
         _p, _p, _p, _p, _p, _i32, _i32, _p, _sz, _p, _p],
    ),
    "hsrq_graph_launch": (_i64, [_p, _p]),
    "hsrq_graph_destroy": (None, [_p]),
    "hsrq_host_workspace_bytes": (_sz, [_i64, _i32, _i64, _i64]),
    "hsrq_solve_group_host": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _p, _p,
         _i32, _i32, _p, _sz, _p],
    ),
    "hsrq_solve_group_host_async": (
        _i64,
        [_p, _i64, _i64, _i32, _p, _p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _p, _p, _p,
         _i32, _i32, _p, _sz, _p],
    ),
    "hsrq_host_wait": (_i64, [_i64]),
    "hsrq_last_launch_count": (_i64, []),
    "hsrq_set_timing": (None, [_i32]),
    "hsrq_tune_diag": (_i32, [_i32, _i32, _i32, _i32, _i32]),
    "hsrq_tune_diag_rx": (_i32, [_i32]),
    "hsrq_tune_panel": (_i32, [_i32]),
    "hsrq_phase_times": (None, [_p]),
    "hsrq_tile_diag": (
        _i64,
        [_i32, _i32, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _f64, _p],
    ),
    "hsrq_tile_update": (
        _i64, [_i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _p, _p, _p, _i32,
               _f64, _p]),
    "hsrq_tile_backtransform": (
        _i64, [_i64, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _i32, _f64, _p]),
    "hsrq_protect_update_batch": (_i64, [_p, _p, _p, _f64, _i64, _p, _p]),
    "hsrq_protect_update_pair_batch": (_i64, [_p, _p, _p, _p, _p, _f64, _i64, _p, _p, _p]),
    "hsrq_hypot_batch": (_i64, [_p, _p, _i64, _p, _p]),
    "hsrq_debug_counters": (_i64, [_p, _i32]),
    "hsrq_debug_stepprof": (_i64, [_p, _i32]),
    "hsrq_compact_encode": (_i64, [_i64, _i32, _p, _p, _p, _p, _p, _p]),
    "hsrq_compact_decode": (_i64, [_i64, _i32, _p, _p, _p, _p, _p, _p]),
    "hsrq_hessenberg_workspace_bytes": (_sz, [_i64]),
    "hsrq_hessenberg_reduce": (_i64, [_p, _i64, _p, _i64, _i64, _p, _sz, _p]),
    "hsrq_backmultiply": (_i64, [_p, _i64, _i64, _p, _i64, _i64, _p, _i64, _p]),
    "hsrq_hessenberg_last_error": (ctypes.c_char_p, []),
    "hsrq_dgemm": (_i64, [_i32, _i32, _i64, _i64, _i64, _f64, _p, _i64, _p, _i64, _f64, _p, _i64, _p]),
    "hsrq_henry_workspace_bytes": (_sz, [_i64, _i64, _i32]),
    "hsrq_henry_solve": (_i64, [_p, _i64, _i64, _p, _i64, _i32, _p, _i64, _p, _p, _sz, _p]),
    "hsrq_h_upload": (_i64, [_p, _i32, _i64, _p, _i64, _p, _p]),
    "hsrq_pack_download": (_i64, [_p, _i64, _i64, _i64, _p, _p, _p, _i32, _p, _p]),
    "hsrq_host_prefault": (_i64, [_p, _i64, _i32]),
}

_lib = None


def load(auto_build=True):
    """Load (building first if the sources are newer) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    path = LIB
    if os.environ.get("HSRQ_LIB_VARIANT"):  # diagnostics build (tools/profile_solve.py)
        path = variant_lib(os.environ["HSRQ_LIB_VARIANT"])
    elif auto_build and stale():
        build()
    if not os.path.exists(path):
        raise ImportError(f"{os.path.basename(path)} not built ({path}); run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def last_error():
    return load().hsrq_last_error().decode()
