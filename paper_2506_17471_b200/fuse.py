"""Fused multi-operator actions (the follow-on of PAPER.md:2477-2482), through libfemgpu's C-ABI
(csrc/fuse.cpp, femgpu_problem_fuse).

Problems on the same cells, geometry and quadrature become one problem whose output is the
concatenation of theirs.  Trial spaces with the same map and input are merged (terms united), so
shared trial values are gathered and evaluated once per cell; the kernels skip the all-zero blocks
of the block-diagonal Psi.

    fused, offsets = fuse_problems([stiffness, mass])
    y = gpu_action(fused)
    y_stiffness, y_mass = split_output(y, offsets)
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import abi
from ._native import lib
from .action import _call
from .form import ProblemInstance
from .io import problem_from_desc


def fuse_problems(problems: Sequence[ProblemInstance]) -> Tuple[ProblemInstance, List[int]]:
    """The fused problem and the row offsets of each problem's output (len(problems) + 1 entries)."""
    n = len(problems)
    cps = [p.to_c() for p in problems]  # keep the flat descriptors (and their arrays) alive
    arr = (C.POINTER(abi.Problem) * n)(*[C.pointer(cp.desc) for cp in cps])
    h = C.c_void_p()
    view = C.POINTER(abi.Problem)()
    offs = (C.c_int64 * (n + 1))()
    _call(lib().femgpu_problem_fuse(arr, n, C.byref(h), C.byref(view), offs))
    try:
        fused = problem_from_desc(view.contents)
    finally:
        lib().femgpu_problem_free(h)
    return fused, [int(o) for o in offs]


def split_output(y: np.ndarray, offsets: Sequence[int]) -> List[np.ndarray]:
    """The per-problem outputs of a fused action."""
    return [y[offsets[i]:offsets[i + 1]] for i in range(len(offsets) - 1)]
