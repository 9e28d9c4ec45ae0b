"""ctypes binding of the C-ABI (include/nextdoor_b200.h).

The product path has no CPU fallback: if libnextdoor_b200.so is missing or
no CUDA device is visible, every engine entry raises.  Status codes map to
the reference's exceptions (SamplerStallError, ValueError, ...).
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, EmptyGraphError, SamplerStallError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnextdoor_b200.so")

ND_OK, ND_ERR_STALL, ND_ERR_APP, ND_ERR_ARG, ND_ERR_CUDA, ND_ERR_NOMEM, ND_ERR_EMPTY = range(7)
ND_SP, ND_TP = 0, 1
(F_FINAL_OFF, F_FINAL_IDS, F_ROOTS, F_ROOTS_OFF, F_CHAIN_LEN, F_STEP_COUNTS, F_STEP_VALS,
 F_REC_COUNTS, F_REC_T, F_REC_V, F_STATS, F_CHAIN_VALS, F_FINAL_IDS32, F_STEP_VALS32) = range(14)
FIELD_DTYPE = {F_FINAL_IDS32: "int32", F_STEP_VALS32: "int32"}  # every other field is int64

vp, i64, u64, i32, u32, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_uint32, C.c_double
pp = C.POINTER(C.c_void_p)
pi64 = C.POINTER(C.c_int64)

# name -> argtypes (all return int unless listed in _RESTYPE)
SIGNATURES = {
    "nd_last_error": [],
    "nd_version": [],
    "nd_copy": [vp, vp, i64, vp],
    "nd_segmented_prefix_sum": [vp, vp, i64, vp, vp],
    "nd_segment_max": [vp, vp, i64, vp, vp],
    "nd_individual_batch": [i32, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, u64, i64,
                            vp, vp],
    "nd_mod_u64": [vp, vp, i64, vp, vp],
    "nd_keyed_u64": [u64, vp, i64, vp, vp, i64, i64, i64, vp, vp],
    "nd_graph_create": [vp, vp, vp, vp, vp, i64, i64, i32, vp, pp],
    "nd_graph_from_edges": [vp, vp, vp, i64, i64, vp, pp],
    "nd_graph_rmat": [i32, i64, u32, u32, u32, u64, i32, i32, vp, pp],
    "nd_text_parse": [C.c_char_p, i64, i32, dbl, dbl, u64, vp, pp, pi64],
    "nd_text_parse_device": [vp, i64, i32, dbl, dbl, u64, vp, pp, pi64],
    "nd_text_host_lines": [vp, vp],
    "nd_text_line_bounds": [vp, i64, pi64],
    "nd_text_finish": [vp, vp, vp, vp, vp, vp, i64, i32, vp, pp, pi64],
    "nd_text_remap": [vp, vp],
    "nd_text_destroy": [vp],
    "nd_graph_destroy": [vp],
    "nd_graph_create_mapped": [vp, vp, vp, vp, i64, i64, vp, pp],
    "nd_graph_build_index": [vp, i32, vp],
    "nd_graph_info": [vp, pi64, pi64, C.POINTER(C.c_int), pi64],
    "nd_graph_footprint": [vp, pi64, pi64, C.POINTER(C.c_double), C.POINTER(C.c_int),
                           C.POINTER(C.c_int)],
    "nd_graph_arrays": [vp, pp, pp, pp, pp, pp],
    "nd_uniform_roots": [vp, i64, u64, i64, i64, vp, vp],
    "nd_run_walk": [vp, i32, vp, i64, i64, i64, vp, i64, u64, i64, i64, i32, vp, pp],
    "nd_run_individual": [vp, i32, vp, i64, vp, i64, i64, i64, vp, i64, u64, i64, i32, vp, i64, vp,
                          pp],
    "nd_run_collective": [vp, i32, i64, i64, i32, i64, i64, i64, i64, i64, i64, vp, vp, u64, i64,
                          vp, i64, vp, pp],
    "nd_transit_schedule": [vp, i64, i64, vp, vp, vp, vp, vp, pi64, vp],
    "nd_result_info": [vp, pi64, pi64, pi64, pi64],
    "nd_result_field": [vp, i32, pp, pi64],
    "nd_result_counters": [vp, pi64, i64],
    "nd_result_copy": [vp, i32, vp, vp],
    "nd_result_narrow_ids": [vp, vp],
    "nd_result_max_row": [vp, pi64],
    "nd_result_dense": [vp, i64, vp, vp],
    "nd_result_profile": [vp, C.POINTER(C.c_double), i64],
    "nd_result_step_times": [vp, C.POINTER(C.c_double), C.POINTER(C.c_double), i64, pi64],
    "nd_set_profiling": [i32],
    "nd_set_concurrency": [i32],
    "nd_format_rows": [vp, vp, i32, vp, i64, vp, vp, vp, i64, pi64],
    "nd_pool_trim": [i64],
    "nd_gather_ceiling": [i64, i32, i32, C.POINTER(C.c_double), vp],
    "nd_result_destroy": [vp],
    "nd_ooc_graph_create": [vp, vp, vp, i64, i64, i64, i32, vp, pp],
    "nd_khop_plan_create": [vp, vp, i64, i64, vp, pp],
    "nd_khop_plan_run": [vp, vp, i64, C.c_uint64, vp],
    "nd_khop_plan_outputs": [vp, pp, pp, pp, pi64, pp, pi64, i64],
    "nd_khop_plan_destroy": [vp],
    "nd_ooc_graph_destroy": [vp],
    "nd_ooc_graph_info": [vp, pi64, pi64, pi64, pi64, pi64],
    "nd_ooc_graph_parts": [vp, vp, i64],
    "nd_run_walk_ooc": [vp, i32, vp, i64, i64, i64, vp, C.c_uint64, i64, vp, pp],
    "nd_run_individual_ooc": [vp, i32, vp, i64, i64, i64, vp, C.c_uint64, vp, pp],
}
_RESTYPE = {"nd_last_error": C.c_char_p}

_lib = None


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python -m paper_2009_06693_b200.build` "
                "(nvcc, sm_100a); the engine has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def last_error() -> str:
    return load().nd_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == ND_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == ND_ERR_STALL:
        raise SamplerStallError("rejection sampler exceeded 1000000 tries")
    if rc == ND_ERR_APP:
        raise ValueError("unknown app code")
    if rc == ND_ERR_ARG:
        raise ValueError(f"invalid argument ({msg})")
    if rc == ND_ERR_NOMEM:
        raise MemoryError(f"device allocation failed ({msg})")
    if rc == ND_ERR_EMPTY:
        raise EmptyGraphError(what or "no edges found")
    raise DeviceError(f"CUDA error ({msg})")


def require_cuda():
    """The engine runs on a CUDA device only; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 engine has no CPU fallback")
    load()
    return torch


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    """Device/host pointer of a contiguous torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        assert t.is_contiguous()
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)
