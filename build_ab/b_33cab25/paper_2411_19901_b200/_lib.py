"""ctypes binding of libslpa_b200.so (include/slpa.h).

The product path has no CPU fallback: if the shared library is missing or no
B200 is visible, every call raises.  Status codes map to the reference's
exception types (ValueError for config / argument errors, RuntimeError for
CUDA failures), see include/slpa.h.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SLPA_LIB: alternative build of the same ABI (A/B timing experiments only).
LIB_PATH = os.environ.get("SLPA_LIB") or os.path.join(HERE, "libslpa_b200.so")

SLPA_OK, SLPA_EINVAL, SLPA_ECUDA, SLPA_EUNSUPPORTED, SLPA_ENOGRAPH, SLPA_EHOOK = range(6)

HOOK_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                           ctypes.POINTER(ctypes.c_int32))


class SlpaConfig(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("scan_mode", ctypes.c_int32),
        ("sketch_slots", ctypes.c_int32),
        ("pickless_gap", ctypes.c_int32),
        ("tolerance", ctypes.c_double),
        ("max_iterations", ctypes.c_int32),
        ("degree_threshold", ctypes.c_int32),
        ("partial_groups", ctypes.c_int32),
        ("worker_count", ctypes.c_int32),
        ("shared_sketch", ctypes.c_int32),
    ]


class SlpaRunStats(ctypes.Structure):
    _fields_ = [
        ("sweeps", ctypes.c_int64),
        ("rounds", ctypes.c_int64),
        ("vertex_evals", ctypes.c_int64),
        ("arc_reads", ctypes.c_int64),
        ("first_evals", ctypes.c_int64),
        ("first_arcs", ctypes.c_int64),
        ("device_ms", ctypes.c_double),
        ("device_bytes", ctypes.c_int64),
        ("graph_bytes", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
    ]


PROF_N = 12
PROF_CLASSES = ("eval_lo_r0", "eval_mid_r0", "eval_hi_r0", "eval_lo_rk", "eval_mid_rk", "eval_hi_rk", "compact",
                "commit", "other", "eval_giant", "unused", "unused")


class SlpaProfile(ctypes.Structure):
    _fields_ = [
        ("launches", ctypes.c_int64 * PROF_N),
        ("ms", ctypes.c_double * PROF_N),
        ("evals", ctypes.c_int64 * PROF_N),
        ("arcs", ctypes.c_int64 * PROF_N),
    ]


# name -> (restype, argtypes); every symbol include/slpa.h declares.
_vp, _i32, _i64, _u32, _u64, _d = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                   ctypes.c_uint64, ctypes.c_double)
SIGNATURES = {
    "slpa_create": (_i32, [_i32, ctypes.POINTER(_vp)]),
    "slpa_destroy": (_i32, [_vp]),
    "slpa_last_error": (ctypes.c_char_p, [_vp]),
    "slpa_version": (ctypes.c_char_p, []),
    "slpa_stream": (_i32, [_vp, ctypes.POINTER(_u64)]),
    "slpa_graph_upload": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    "slpa_graph_upload_device": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp]),
    "slpa_graph_set_order": (_i32, [_vp, _vp]),
    "slpa_graph_info": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                               ctypes.POINTER(_i32)]),
    "slpa_graph_download": (_i32, [_vp, _vp, _vp, _vp]),
    "slpa_gen_rmat": (_i32, [_vp, _i32, _i64, _u32, _u32, _u32, _u64, _i32, _u64]),
    "slpa_gen_grid": (_i32, [_vp, _i64, _i64, _i32, _u64]),
    "slpa_gen_kmer": (_i32, [_vp, _i64, _u32, _u64, _i32, _u64]),
    "slpa_build_graph": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _i32]),
    "slpa_run": (_i32, [_vp, ctypes.POINTER(SlpaConfig), _vp, _vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                        HOOK_FN, _vp]),
    "slpa_move": (_i32, [_vp, ctypes.POINTER(SlpaConfig), _vp, _vp, _i32, ctypes.POINTER(_i64)]),
    "slpa_get_labels": (_i32, [_vp, _vp]),
    "slpa_last_run_stats": (_i32, [_vp, ctypes.POINTER(SlpaRunStats)]),
    "slpa_set_profiling": (_i32, [_vp, _i32]),
    "slpa_get_profile": (_i32, [_vp, ctypes.POINTER(SlpaProfile)]),
    "slpa_aux_memory_estimate": (_i64, [_i64, _i32, ctypes.POINTER(SlpaConfig)]),
    "slpa_modularity": (_i32, [_vp, _vp, ctypes.POINTER(_d), ctypes.POINTER(_i64), _vp, _vp, _vp]),
    "slpa_part_upload": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i32]),
    "slpa_part_gen_rmat": (_i32, [_vp, _i32, _i64, _u32, _u32, _u32, _u64, _i32, _u64, _i64, _i64]),
    "slpa_part_info": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                              ctypes.POINTER(_i64)]),
    "slpa_part_buffers": (_i32, [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "slpa_rmat_cuts": (_i32, [_vp, _i32, _i64, _u32, _u32, _u32, _u64, _i32, _u64, _i32, _vp]),
    "slpa_part_arc_hash": (_i32, [_vp, _vp]),
    "slpa_part_set_symmetric": (_i32, [_vp, _i32]),
    "slpa_part_begin": (_i32, [_vp, ctypes.POINTER(SlpaConfig)]),
    "slpa_part_sweep": (_i32, [_vp, ctypes.POINTER(SlpaConfig), _i32, ctypes.POINTER(_i64)]),
    "slpa_part_end_exchange": (_i32, [_vp]),
    "slpa_part_det_buffers": (_i32, [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "slpa_part_det_round": (_i32, [_vp, ctypes.POINTER(SlpaConfig), _i32, _i32]),
    "slpa_part_det_import": (_i32, [_vp, ctypes.POINTER(_i64)]),
    "slpa_part_det_commit": (_i32, [_vp, ctypes.POINTER(SlpaConfig), ctypes.POINTER(_i64)]),
    "slpa_part_tally": (_i32, [_vp, ctypes.POINTER(_d), ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "slpa_part_modularity": (_i32, [_vp, _d, ctypes.POINTER(_d)]),
    "slpa_validate_graph": (_i32, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_d),
                                   ctypes.POINTER(_d)]),
    "slpa_edges_parse": (_i32, [ctypes.c_char_p, _i32, _i32, ctypes.POINTER(_vp)]),
    "slpa_edges_info": (_i32, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                               ctypes.POINTER(_i32), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                               ctypes.POINTER(_i64)]),
    "slpa_edges_copy": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "slpa_edges_free": (None, [_vp]),
    "slpa_format_count": (_i64, [_i64, _vp, _vp, _i32]),
    "slpa_format_rows": (_i32, [_i64, _i64, _vp, _vp, _vp, _i32, _i32, _i32, ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(_i64)]),
    "slpa_free_buffer": (None, [_vp]),
}

_LIB = None
_LOCK = threading.Lock()


def load_library(path: str | None = None):
    """Load (once) and return the CDLL; raises if the .so is absent."""
    global _LIB
    with _LOCK:
        if _LIB is not None and path is None:
            return _LIB
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"{p} is not built; run `python -m paper_2411_19901_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _LIB = lib
        return lib


class SlpaError(RuntimeError):
    pass


def check(lib, ctx, code: int):
    if code == SLPA_OK:
        return
    msg = lib.slpa_last_error(ctx)
    msg = msg.decode() if msg else f"slpa error {code}"
    if code in (SLPA_EINVAL, SLPA_EUNSUPPORTED):
        raise ValueError(msg)
    raise SlpaError(msg)
