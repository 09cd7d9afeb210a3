"""Instance and candidate files in the reference's versioned structured-text format
(femsched io.hpp, format_version 1), through libfemgpu's C-ABI (csrc/io.cpp):

  save_instance / load_instance    femsched::save_instance_file / load_instance_file (io.hpp:381-391)
  save_schedule / load_schedule    femsched::save_candidate / load_candidate (io.hpp:407-460)

Doubles carry 17 significant digits, so a round trip is bit-exact and the text is byte-identical
to the reference writer's."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from ._native import lib
from .action import TilingParams, _call
from .form import (FormSignature, IndexMap, MeshConnectivity, PointwiseMap, ProblemInstance, ScalarSpace,
                   Tabulations, VectorSpace)


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def problem_from_desc(d: abi.Problem) -> ProblemInstance:
    """Copies a flat femgpu_problem descriptor into the host data model (form.py)."""
    Q = d.quad_points
    sig = FormSignature(dim=d.dim, quad_points=Q, coord_dofs=d.coord_dofs,
                        affine_geometry=bool(d.affine_geometry), coordinate_space=d.coordinate_space,
                        word_bytes=d.word_bytes, test_dofs=d.test_dofs, test_deriv_terms=d.test_deriv_terms)
    tab = Tabulations()
    conn = MeshConnectivity(cell_count=d.cell_count)
    sx, vx = [], []
    for i in range(d.n_scalar):
        s = d.scalar_spaces[i]
        sig.scalar_spaces.append(ScalarSpace(s.dofs, s.deriv_terms))
        tab.scalar_phi.append(_arr(s.phi, s.deriv_terms * Q * s.dofs, np.float64).reshape(s.deriv_terms, Q, s.dofs))
        conn.scalar_maps.append(IndexMap(_arr(s.map, d.cell_count * s.dofs, np.int32).reshape(d.cell_count, s.dofs),
                                         s.global_count))
        sx.append(_arr(s.input, s.global_count, np.float64))
    for i in range(d.n_vector):
        s = d.vector_spaces[i]
        comps = [int(c) for c in _arr(s.components, s.deriv_terms, np.int32)]
        sig.vector_spaces.append(VectorSpace(s.dofs, s.deriv_terms, comps))
        tab.vector_phi.append(_arr(s.phi, s.deriv_terms * Q * s.dofs, np.float64).reshape(s.deriv_terms, Q, s.dofs))
        conn.vector_maps.append(IndexMap(_arr(s.map, d.cell_count * s.dofs, np.int32).reshape(d.cell_count, s.dofs),
                                         s.global_count))
        vx.append(_arr(s.input, s.global_count * d.dim, np.float64))
    tab.psi = _arr(d.psi, d.test_deriv_terms * d.test_dofs * Q, np.float64).reshape(d.test_deriv_terms, d.test_dofs, Q)
    tab.weights = _arr(d.weights, Q, np.float64)
    conn.test_map = IndexMap(_arr(d.test_map, d.cell_count * d.test_dofs, np.int32).reshape(d.cell_count, d.test_dofs),
                             d.test_global_count)
    if d.affine_geometry:
        conn.coord_map = IndexMap(_arr(d.coord_map, d.cell_count * d.coord_dofs, np.int32)
                                  .reshape(d.cell_count, d.coord_dofs), d.coord_global_count)
        conn.coord_global_count = d.coord_global_count
        conn.coords = _arr(d.coords, d.coord_global_count * d.dim, np.float64).reshape(d.coord_global_count, d.dim)
    m = PointwiseMap()
    for i in range(d.n_map_nodes):
        n = d.map_nodes[i]
        m.nodes.append((int(n.op), float(n.value), int(n.a), int(n.b)))
    m.outputs = [int(x) for x in _arr(d.map_outputs, d.n_map_outputs, np.int32)]
    return ProblemInstance(sig, m, tab, conn, sx, vx, d.output_size)


def save_instance(problem: ProblemInstance, path: str) -> None:
    """femsched::save_instance_file (io.hpp:381-385)."""
    cp = problem.to_c()
    _call(lib().femgpu_problem_save(C.byref(cp.desc), str(path).encode()))


def load_instance(path: str) -> ProblemInstance:
    """femsched::load_instance_file (io.hpp:387-391): validated on load."""
    h = C.c_void_p()
    view = C.POINTER(abi.Problem)()
    _call(lib().femgpu_problem_load(str(path).encode(), C.byref(h), C.byref(view)))
    try:
        return problem_from_desc(view.contents)
    finally:
        lib().femgpu_problem_free(h)


def save_schedule(params: TilingParams, path: str, n_scalar: int = 0, n_vector: int = 0) -> None:
    """femsched::save_candidate (io.hpp:407-428); B200 kinds as extension kinds."""
    s = params.to_c()
    n_scalar = max(n_scalar, len(params.eval_col_tiles_scalar))
    n_vector = max(n_vector, len(params.eval_col_tiles_vector))
    _call(lib().femgpu_schedule_save(C.byref(s), n_scalar, n_vector, str(path).encode()))


def load_schedule(path: str) -> TilingParams:
    """femsched::load_candidate (io.hpp:430-455)."""
    s = abi.Schedule()
    _call(lib().femgpu_schedule_load(str(path).encode(), C.byref(s)))
    return TilingParams.from_c(s)
