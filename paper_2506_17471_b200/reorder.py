"""Locality-restoring renumbering of a general mesh (csrc/reorder.cpp, femgpu_problem_reorder).

    q, perms = reorder_problem(p)          # q = p with cells in Morton order, nodes first-touch
    y_q = gpu_action(q)
    y_p = np.empty_like(y_q); y_p[perms["output"]] = y_q    # back to p's row numbering
    x_q = x_p[perms["scalar"][0]]                            # a later input of scalar space 0

Every perm maps new -> old.  The action of q is the action of p permuted, up to the floating-point
order of the per-row sums.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Tuple

import numpy as np

from . import abi
from ._native import lib
from .action import _call
from .form import ProblemInstance
from .io import problem_from_desc


def reorder_problem(p: ProblemInstance) -> Tuple[ProblemInstance, Dict[str, object]]:
    cp = p.to_c()
    cells = p.connectivity.cell_count
    cell_perm = np.empty(cells, dtype=np.int32)
    out_perm = np.empty(p.output_size, dtype=np.int32)
    sp = [np.empty(m.global_count, dtype=np.int32) for m in p.connectivity.scalar_maps]
    vp = [np.empty(m.global_count, dtype=np.int32) for m in p.connectivity.vector_maps]
    iptr = C.POINTER(C.c_int32)
    sarr = (iptr * max(1, len(sp)))(*[a.ctypes.data_as(iptr) for a in sp])
    varr = (iptr * max(1, len(vp)))(*[a.ctypes.data_as(iptr) for a in vp])
    h = C.c_void_p()
    view = C.POINTER(abi.Problem)()
    _call(lib().femgpu_problem_reorder(C.byref(cp.desc), C.byref(h), C.byref(view), cell_perm.ctypes.data_as(iptr),
                                       out_perm.ctypes.data_as(iptr), sarr, varr))
    try:
        q = problem_from_desc(view.contents)
    finally:
        lib().femgpu_problem_free(h)
    return q, {"cells": cell_perm, "output": out_perm, "scalar": sp, "vector": vp}


def output_to_original(y_new: np.ndarray, perms: Dict[str, object]) -> np.ndarray:
    """y in the original row numbering."""
    y = np.empty_like(y_new)
    y[perms["output"]] = y_new
    return y


def inputs_to_new(xs: List[np.ndarray], vs: List[np.ndarray], perms: Dict[str, object], dim: int):
    """Later inputs (original numbering) in the reordered numbering."""
    return ([x[perm] for x, perm in zip(xs, perms["scalar"])],
            [v.reshape(-1, dim)[perm].reshape(-1) for v, perm in zip(vs, perms["vector"])])
