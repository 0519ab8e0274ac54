"""Loader for the in-tree CUDA library libmrlbm_b200.so (built by build.py).

Fails loudly when the library is missing: there is no CPU fallback in the
product path.
"""
import ctypes as C
import os

from .abi import SchemeSpec, RunConfig, StepStats, TieRecord

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmrlbm_b200.so")
_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "mrlbm_create": (C.c_int, [P(SchemeSpec), P(RunConfig), P(vp)]),
        "mrlbm_load_leaves": (C.c_int, [vp, C.c_int, C.c_int64, vp, vp]),
        "mrlbm_commit": (C.c_int, [vp]),
        "mrlbm_step": (C.c_int, [vp, C.c_int, P(StepStats)]),
        "mrlbm_level_count": (C.c_int, [vp, C.c_int, P(C.c_int64)]),
        "mrlbm_read_leaves": (C.c_int, [vp, C.c_int, vp, vp]),
        "mrlbm_set_profiling": (C.c_int, [vp, C.c_int]),
        "mrlbm_tie_log": (C.c_int, [vp, P(TieRecord), C.c_int, P(C.c_int64), C.c_int]),
        "mrlbm_set_graph": (C.c_int, [vp, C.c_int]),
        "mrlbm_profile_text": (C.c_int, [vp, C.c_char_p, C.c_int, C.c_int]),
        "mrlbm_stream_handle": (vp, [vp]),
        "mrlbm_synchronize": (C.c_int, [vp]),
        "mrlbm_last_error": (C.c_char_p, [vp]),
        "mrlbm_destroy": (None, [vp]),
        "mrlbm_finest_count": (C.c_int, [vp, P(C.c_int64)]),
        "mrlbm_reconstruct_finest": (C.c_int, [vp, vp]),
        "mrlbm_additional_error": (C.c_int, [vp, vp, vp, P(C.c_double), vp]),
        "mrlbm_stream_table": (C.c_int, [C.c_int, C.c_int, P(C.c_int32), C.c_int, C.c_int, vp, vp, P(C.c_int)]),
        "mrlbm_build_config": (C.c_int, [C.c_int, C.c_int, C.c_double, P(SchemeSpec), P(RunConfig)]),
        "mrlbm_config_steps": (C.c_int64, [C.c_int, P(RunConfig)]),
        "mrlbm_initial_finest": (C.c_int, [C.c_int, P(SchemeSpec), P(RunConfig), C.c_uint64, vp]),
        "mrlbm_set_force_tracking": (C.c_int, [vp, C.c_int]),
        "mrlbm_force_history": (C.c_int, [vp, vp, vp, C.c_int, P(C.c_int)]),
        "mrlbm_drag_lift": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                      P(C.c_double), P(C.c_double)]),
        "mrlbm_strouhal": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double,
                                     P(C.c_double), P(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
