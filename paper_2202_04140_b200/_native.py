"""ctypes binding of the C ABI in include/acedag_b200.h.

The library ``libacedag_b200.so`` is built in-tree by ``build.py`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing, importing the evaluator raises, and every numeric call
goes through the CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libacedag_b200.so")

OK, EINVAL, EMISSING_SEED, ECUDA, ENOMEM, ENOTTARGET, EDOMAIN, EUNSUPPORTED, EFORMAT = 0, -1, -2, -3, -4, -5, -6, -7, -8
METHOD_RECURSIVE, METHOD_NAIVE = 0, 1
OUT_REAL, OUT_COMPLEX = 0, 1
PREC_F64, PREC_F32 = 0, 1

_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_dp = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol of include/acedag_b200.h
SIGNATURES = {
    "acedag_abi_version": (C.c_int, []),
    "acedag_last_error": (C.c_char_p, []),
    "acedag_graph_build": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "acedag_graph_from_parents": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                            C.c_int64, C.c_int64, _i32p, _u8p, C.POINTER(_vp)]),
    "acedag_graph_destroy": (None, [_vp]),
    "acedag_graph_info": (C.c_int, [_vp, _i64p, _i64p, _i64p, _i64p, _i32p]),
    "acedag_graph_arrays": (C.c_int, [_vp, _i32p, _u8p, _i32p, _i32p]),
    "acedag_graph_node_seeds": (C.c_int, [_vp, C.c_int64, _i32p, C.c_int32]),
    "acedag_graph_find": (C.c_int64, [_vp, _i32p, C.c_int32]),
    "acedag_graph_serialize": (C.c_int, [_vp, C.c_char_p, _i64p]),
    "acedag_graph_deserialize": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(_vp), _i32p, _i64p, _i64p, _i64p]),
    "acedag_graph_spec": (C.c_int, [_vp, _i32p, _i32p, _dp, _i32p, _i32p, _i32p]),
    "acedag_plan_create": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "acedag_plan_destroy": (None, [_vp]),
    "acedag_plan_set_coefficients": (C.c_int, [_vp, _i64p, _dp, _dp, C.c_int64, C.c_int32]),
    "acedag_plan_program": (C.c_int, [_vp, _i64p, _dp, _dp, C.c_int64, C.c_int32, C.c_int32, _vp, _i64p,
                                       _vp, _i64p, _i32p, _i64p]),
    "acedag_plan_program_horner": (C.c_int, [_vp, _i64p, _dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _vp,
                                              _i64p, _i32p, _i32p]),
    "acedag_plan_info": (C.c_int, [_vp, _i64p, _i64p, _i64p, _i64p]),
    "acedag_eval": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp]),
    "acedag_eval_kernel_name": (C.c_char_p, [_vp, C.c_int, C.c_int, C.c_int, C.c_int64]),
    "acedag_naive_products": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, _vp]),
    "acedag_reduce_sites": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "acedag_eval_nodes": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "acedag_pool": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_int64, C.c_int32, _vp, _vp]),
    "acedag_check_coords": (C.c_int, [C.c_int, _dp, C.c_int64]),
    "acedag_pool_positions": (C.c_int, [C.c_int, _vp, _vp, C.c_int64, C.c_int32, C.c_double, C.c_double,
                                        _vp, _vp]),
    "acedag_launch_count": (C.c_int64, []),
    "acedag_plan_timing": (C.c_int, [_vp, C.c_int]),
    "acedag_plan_timing_read": (C.c_int, [_vp, _vp, _vp]),
    "acedag_eval_host": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int64, _vp, _vp, _vp]),
    "acedag_eval_from_positions": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_double, C.c_double,
                                             C.c_int, _vp, _vp]),
}


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lib = None


def lib():
    """Load the in-tree CUDA library; raise loudly when it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def last_error() -> str:
    return lib().acedag_last_error().decode("utf-8", "replace")


def check(rc: int) -> int:
    """Map a C status onto the reference's exception types."""
    if rc >= 0:
        return rc
    msg = last_error()
    if rc in (EINVAL, ENOTTARGET, EDOMAIN):
        raise ValueError(msg)
    if rc == EMISSING_SEED:
        raise KeyError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise NativeError(rc, msg)


def ptr(arr, ctype):
    """ctypes pointer to a contiguous numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))
