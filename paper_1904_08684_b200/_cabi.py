"""ctypes binding of ``libqfswe.so`` (the C ABI declared in include/qfswe.h).

This is the thin layer the reference package would add to call the B200
path.  Loading fails loudly when the library is missing or
no CUDA device is present: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# QF_LIB: diagnostic override (tools/variants.py builds knob variants there)
LIB_PATH = Path(os.environ.get("QF_LIB") or Path(__file__).resolve().parent / "_lib" / "libqfswe.so")

QF_OK, QF_E_DRY, QF_E_SINGULAR, QF_E_NONFINITE, QF_E_CUDA, QF_E_ARG = range(6)
BIT_DRY, BIT_SINGULAR, BIT_NONFINITE = 1, 2, 4
TERM_VOLUME, TERM_EDGE, TERM_SOURCE, TERM_ALL = 1, 2, 4, 7

EXPORTS = (
    "qf_create", "qf_destroy", "qf_velocity", "qf_static", "qf_project", "qf_ghost", "qf_rhs", "qf_stage", "qf_step",
    "qf_run", "qf_pack", "qf_unpack", "qf_gather", "qf_scatter", "qf_error", "qf_fill", "qf_l2_error", "qf_rhs_mass",
    "qf_stage_push", "qf_signal", "qf_wait", "qf_ipc_export", "qf_ipc_import", "qf_ipc_close_all",
    "qf_launch_count", "qf_last_error", "qf_abi_version", "qf_stage_events", "qf_rhs_ex", "qf_user_scenario", "qf_halo_traces", "qf_halo_table", "qf_copy", "qf_ghost_dev", "qf_advance_time",
    "qf_graph_begin", "qf_graph_end", "qf_graph_launch", "qf_graph_destroy",
)


class QfDesc(C.Structure):
    _fields_ = [
        ("order", C.c_int32), ("n_elem", C.c_int32), ("ld", C.c_int64),
        ("geo", C.c_void_p), ("hb", C.c_void_p), ("nbr", C.c_void_p),
        ("n_bnd", C.c_int32), ("bnd_elem", C.c_void_p), ("bnd_local", C.c_void_p),
        ("ghost", C.c_void_p), ("hbt", C.c_void_p),
        ("g", C.c_double), ("f_c", C.c_double), ("tau_bf", C.c_double),
        ("hb_linear", C.c_int32), ("scn_kind", C.c_int32), ("scn_params", C.c_double * 8),
        ("has_forcing", C.c_int32), ("taylor", C.c_int32), ("block", C.c_int32),
        ("uni", C.c_void_p),
    ]


_lib = None


def load(path: Path | None = None):
    """Load the library and declare signatures (no CUDA call is made)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path or LIB_PATH)
    if not p.exists():
        raise RuntimeError(f"{p} not built: run `python -m paper_1904_08684_b200.build`")
    lib = C.CDLL(str(p))
    vp, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "qf_create": (C.c_int, [C.POINTER(QfDesc), C.POINTER(C.c_void_p)]),
        "qf_destroy": (None, [vp]),
        "qf_velocity": (C.c_int, [vp, vp, vp, i32, i32, vp]),
        "qf_ghost": (C.c_int, [vp, d, vp]),
        "qf_project": (C.c_int, [vp, vp, i32, d, vp, vp, vp]),
        "qf_static": (C.c_int, [vp, i32, vp]),
        "qf_rhs": (C.c_int, [vp, vp, vp, d, i32, vp, vp, vp]),
        "qf_rhs_mass": (C.c_int, [vp, vp, vp, d, i32, vp, vp, vp, vp]),
        "qf_rhs_ex": (C.c_int, [vp, vp, vp, d, i32, vp, vp, vp, vp, vp]),
        "qf_stage": (C.c_int, [vp, vp, vp, vp, vp, vp, d, d, d, d, vp, d, i32, i32, vp]),
        "qf_step": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "qf_run": (C.c_int, [vp, i32, vp, vp, vp, vp, i32, vp]),
        "qf_pack": (C.c_int, [vp, vp, i32, i32, i32, i64, vp, vp]),
        "qf_unpack": (C.c_int, [vp, vp, i32, i32, i32, i64, vp, vp]),
        "qf_gather": (C.c_int, [vp, i64, vp, i32, i32, vp, vp]),
        "qf_scatter": (C.c_int, [vp, vp, i32, i32, vp, i64, vp]),
        "qf_error": (C.c_int, [vp, C.POINTER(C.c_uint32), i32, vp]),
        "qf_fill": (C.c_int, [vp, C.c_size_t, d, vp]),
        "qf_l2_error": (C.c_int, [vp, vp, d, i32, i32, vp, vp]),
        "qf_stage_push": (C.c_int, [vp, vp, vp, vp, vp, vp, d, d, d, d, vp, d, i32, i32, vp, vp,
                                    vp, vp]),
        "qf_halo_traces": (C.c_int, [vp, vp, vp, vp, i32, vp, vp]),
        "qf_halo_table": (C.c_int, [vp, vp]),
        "qf_copy": (C.c_int, [vp, vp, C.c_size_t, vp]),
        "qf_signal": (C.c_int, [vp, C.c_uint32, vp]),
        "qf_wait": (C.c_int, [vp, C.c_uint32, vp]),
        "qf_ipc_export": (C.c_int, [vp, vp, C.POINTER(C.c_uint64)]),
        "qf_ipc_import": (C.c_int, [vp, C.c_uint64, C.POINTER(C.c_void_p)]),
        "qf_ipc_close_all": (C.c_int, []),
        "qf_launch_count": (C.c_uint64, []),
        "qf_last_error": (C.c_char_p, []),
        "qf_abi_version": (C.c_int, []),
        "qf_stage_events": (C.c_int, [vp, C.POINTER(C.c_void_p), i32]),
        "qf_user_scenario": (C.c_int, [vp, vp, C.c_size_t, i32]),
        "qf_ghost_dev": (C.c_int, [vp, vp, d, vp]),
        "qf_advance_time": (C.c_int, [vp, vp]),
        "qf_graph_begin": (C.c_int, [vp]),
        "qf_graph_end": (C.c_int, [vp, C.POINTER(C.c_void_p)]),
        "qf_graph_launch": (C.c_int, [vp, C.c_uint32, vp]),
        "qf_graph_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("QF_LIB") and not hasattr(lib, name):
            continue  # diagnostic builds of older sources (tools/variants.py)
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status != QF_OK:
        msg = (_lib.qf_last_error() or b"").decode()
        raise RuntimeError(f"{what} failed with status {status}: {msg}")
