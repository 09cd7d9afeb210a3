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


class FusedOperator:
    """The operators of `problems` applied together, fused into one kernel or run separately,
    whichever measures faster on this device (the fused state can cost more registers than the shared
    gathers save: the Stokes pair of mesh.FUSED_PAIRS runs 0.95x fused, Laplace + mass 1.13x).

        op = FusedOperator([stiffness, mass]); y_k, y_m = op.action(); op.close()
    """

    def __init__(self, problems: Sequence[ProblemInstance], choose: bool = True, steps: int = 10):
        from .action import GpuInstance
        self.fused_problem, self.offsets = fuse_problems(problems)
        self._fused = GpuInstance(self.fused_problem)
        self._separate = None
        self.mode = "fused"
        self.times = {}
        if choose:
            self._fused.action()
            self.times["fused"] = self._fused.time_steps(steps, pipelined=True) / steps
            sep = [GpuInstance(p) for p in problems]
            t = 0.0
            for g in sep:
                g.action()
                t += g.time_steps(steps, pipelined=True) / steps
            self.times["separate"] = t
            if t < self.times["fused"]:
                self._fused.close()
                self._fused, self._separate, self.mode = None, sep, "separate"
            else:
                for g in sep:
                    g.close()

    def action(self) -> List[np.ndarray]:
        if self._separate is not None:
            return [g.action() for g in self._separate]
        return split_output(self._fused.action(), self.offsets)

    def close(self):
        for g in ([self._fused] if self._fused else []) + (self._separate or []):
            g.close()
        self._fused, self._separate = None, None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
