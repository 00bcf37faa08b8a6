"""Host view of the compiled recursive program (csrc/plan.cpp) -- no device.

Used by tooling and the CPU test-suite to inspect the per-warp DFS program
the K2 kernel walks: one 16-byte record per product node in preorder.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .graph import as_eval_graph

# {coefficient, byte offset of the seed row (slot * 512), #children, subtree size}
OP_DTYPE = np.dtype([("c", "<f8"), ("off", "<u4"), ("nch", "<u2"), ("skip", "<u2")])
ROW_BYTES = 512


def compile_program(graph, node_ids, values, warps: int = 32) -> dict:
    g = as_eval_graph(graph)
    node_ids = np.ascontiguousarray(np.asarray(node_ids, np.int64).reshape(-1))
    values = np.asarray(values)
    if values.ndim == 1:
        values = values[:, None]
    n_out = values.shape[1]
    c_re = np.ascontiguousarray(values.real, np.float64)
    c_im = np.ascontiguousarray(values.imag, np.float64) if np.iscomplexobj(values) else None
    lib = N.lib()
    ns, no = C.c_int64(), C.c_int64()
    args = (g._h, N.ptr(node_ids, C.c_int64), N.ptr(c_re, C.c_double), N.ptr(c_im, C.c_double),
            node_ids.shape[0], n_out, warps)
    N.check(lib.acedag_plan_program(*args, None, C.byref(ns), None, C.byref(no), None, None))
    slots = np.empty(max(1, ns.value), np.uint16)
    ops = np.empty(max(1, no.value), OP_DTYPE)
    chunk = np.empty(warps + 1, np.int32)
    stats = np.empty(3, np.int64)
    N.check(lib.acedag_plan_program(*args, C.c_void_p(slots.ctypes.data), C.byref(ns),
                                    C.c_void_p(ops.ctypes.data), C.byref(no), N.ptr(chunk, C.c_int32),
                                    N.ptr(stats, C.c_int64)))
    return {"slot_label": slots[: ns.value], "ops": ops[: no.value], "chunk": chunk,
            "recursive_products": int(stats[0]), "extra_nodes": int(stats[1]),
            "naive_products": int(stats[2])}


# k2_horner records (csrc/horner.h): {coefficient, z = class-scaled seed
# offset, w = nch | nhot << 15 | nsm << 22 (a root's second record: class
# flags cls_a | cls_b << 2 | single << 4)}
OPH_DTYPE = np.dtype([("c", "<f8"), ("z", "<u4"), ("w", "<u4")])
HORNER_HOT, HORNER_MAX_LEAVES = 32, 30


def compile_horner(graph, node_ids, values, warps: int = 128, hot: int = HORNER_HOT, us: int = 97) -> dict:
    """The k2_horner encoding of the recursive program (host only): records
    of the four TMEM-lane-quadrant copies [4, n], chunk offsets, roots per
    chunk, and the slot labels of compile_program."""
    g = as_eval_graph(graph)
    node_ids = np.ascontiguousarray(np.asarray(node_ids, np.int64).reshape(-1))
    c_re = np.ascontiguousarray(np.asarray(values, np.float64).reshape(-1))
    lib = N.lib()
    no = C.c_int64()
    args = (g._h, N.ptr(node_ids, C.c_int64), N.ptr(c_re, C.c_double), node_ids.shape[0], warps, hot, us)
    N.check(lib.acedag_plan_program_horner(*args, None, C.byref(no), None, None))
    ops = np.empty(4 * max(1, no.value), OPH_DTYPE)
    chunk = np.empty(warps + 1, np.int32)
    croots = np.empty(warps, np.int32)
    N.check(lib.acedag_plan_program_horner(*args, C.c_void_p(ops.ctypes.data), C.byref(no),
                                           N.ptr(chunk, C.c_int32), N.ptr(croots, C.c_int32)))
    prog = compile_program(graph, node_ids, c_re, warps)
    return {"ops": ops[: 4 * no.value].reshape(4, no.value), "chunk": chunk, "croots": croots,
            "slot_label": prog["slot_label"], "hot": hot, "us": us}
