"""ctypes declarations for libtilelink_b200.so (include/tl_api.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_LIB = None

TL_OK, TL_ERR_INVALID, TL_ERR_UNSUPPORTED, TL_ERR_CUDA, TL_ERR_TIMEOUT, TL_ERR_STATE = range(6)
STATUS_NAMES = ["TL_OK", "TL_ERR_INVALID", "TL_ERR_UNSUPPORTED", "TL_ERR_CUDA", "TL_ERR_TIMEOUT", "TL_ERR_STATE"]

_vp, _i64, _int = C.c_void_p, C.c_int64, C.c_int
_vpp = C.POINTER(C.c_void_p)

SIGNATURES = {
    "tl_status_string": (C.c_char_p, [_int]),
    "tl_last_error": (C.c_char_p, []),
    "tl_build_info": (C.c_char_p, []),
    "tl_handle_size": (C.c_size_t, []),
    "tl_comm_create": (_int, [_int, _int, _int, _i64, _i64, _vp, C.POINTER(_vp)]),
    "tl_comm_connect": (_int, [_vp, _vp]),
    "tl_comm_create_loopback": (_int, [_int, _int, _i64, _i64, C.POINTER(_vp)]),
    "tl_comm_destroy": (_int, [_vp]),
    "tl_comm_info": (_int, [_vp, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)]),
    "tl_set_option": (_int, [_vp, C.c_char_p, _i64]),
    "tl_get_option": (_int, [_vp, C.c_char_p, C.POINTER(_i64)]),
    "tl_comm_check": (_int, [_vp, C.POINTER(_i64)]),
    "tl_ag_gemm": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "tl_ag_gemm_act": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp]),
    "tl_gemm_rs": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "tl_mlp_forward": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _vp]),
    "tl_ag_gemm_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _vpp, _i64, _i64, _i64, _int, _vp]),
    "tl_gemm_rs_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _i64, _i64, _i64, _vp]),
    "tl_mlp_forward_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _vpp, _vpp, _i64, _i64, _i64, _int, _vp]),
    "tl_debug_static_map": (_int, [_i64, _int, _i64, _int, _i64, C.POINTER(_i64)]),
    "tl_moe_capacity": (_i64, [_vp, _i64, _int, _int]),
    "tl_comm_create_ex": (_int, [_int, _int, _int, _i64, _i64, _int, _vp, C.POINTER(_vp)]),
    "tl_comm_create_loopback_ex": (_int, [_int, _int, _i64, _i64, _int, C.POINTER(_vp)]),
    "tl_moe_gemm_rs": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp]),
    "tl_moe_gemm_rs_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _vpp, _vpp, _vpp, _i64, _i64, _i64, _int, _int, _vp]),
    "tl_sp_attention": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _int, _int, C.c_float, _vp]),
    "tl_sp_attention_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _vpp, _i64, _int, _int, C.c_float, _vp]),
    "tl_moe_ag_gemm": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _int, _vp]),
    "tl_moe_ag_gemm_loopback": (_int, [_vp, _vpp, _vpp, _vpp, _vpp, _vpp, _vpp, _i64, _i64, _i64, _int, _int, _int,
                                       _vp]),
    "tl_trace_read": (_int, [_vp, _vp, _i64, C.POINTER(_i64)]),
}


class TLError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{fn}: {name}: {msg}")


def lib(build_if_missing: bool = True):
    """Load the in-tree library (building it first if sources are newer).  Never falls back."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("TL_LIB_PATH", _build.LIB)   # experiments only: A/B of two builds
    if path == _build.LIB and build_if_missing and not _build.up_to_date():
        try:
            _build.build()
        except Exception:
            if not os.path.exists(path):
                raise
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -m paper_2503_20313_b200.build` (nvcc, sm_100a)")
    L = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def check(status: int, fn: str):
    if status != TL_OK:
        raise TLError(status, fn, lib().tl_last_error().decode())


def ptr_array(ptrs):
    arr = (C.c_void_p * len(ptrs))(*[p if p else None for p in ptrs])
    return C.cast(arr, _vpp), arr
