"""TEST INFRASTRUCTURE ONLY — the parity checker.

Loads the two CPU checkers built by oracle/Makefile:
  * liboracle.so              — C restatement of femsched::reference_action (femoracle.c)
  * _ref/libfemsched_ref.so   — the reference's own form.hpp compiled in place (ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
this module.  The product path (paper_2506_17471_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2506_17471_b200 import abi
from paper_2506_17471_b200.form import (FormSignature, IndexMap, MeshConnectivity, PointwiseMap,
                                        ProblemInstance, ScalarSpace, Tabulations, VectorSpace)

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libfemsched_ref.so")

_lib = None
_ref = None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def build():
    """Builds liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE):
            build()
        L = C.CDLL(_ORACLE)
        L.oracle_reference_action_range.argtypes = [C.POINTER(abi.Problem), C.c_int, C.c_int,
                                                    C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                                    C.c_char_p, C.c_int]
        L.oracle_validate.argtypes = [C.POINTER(abi.Problem), C.c_char_p, C.c_int]
        L.oracle_usable_flops.argtypes = [C.POINTER(abi.Problem)]
        L.oracle_usable_flops.restype = C.c_longlong
        L.oracle_uniform_fill.argtypes = [C.POINTER(C.c_uint64), C.c_double, C.c_double,
                                          C.POINTER(C.c_double), C.c_longlong]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            build()
        if not os.path.exists(_REF):
            raise FileNotFoundError("oracle/_ref/libfemsched_ref.so not built (reference sources absent)")
        L = C.CDLL(_REF)
        L.ref_reference_action.argtypes = [C.POINTER(abi.Problem), C.POINTER(C.c_double),
                                           C.POINTER(C.c_longlong), C.c_char_p, C.c_int]
        L.ref_make_preset.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong,
                                      C.c_char_p, C.c_int]
        L.ref_make_preset.restype = C.c_void_p
        L.ref_instance_desc.argtypes = [C.c_void_p]
        L.ref_instance_desc.restype = C.POINTER(abi.Problem)
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_usable_flops.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int]
        L.ref_usable_flops.restype = C.c_longlong
        L.ref_time_threads.argtypes = [C.POINTER(abi.Problem), C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.c_char_p, C.c_int]
        L.ref_time_threads.restype = C.c_double
        _ref = L
    return _ref


def _desc(p):
    return p.to_c() if isinstance(p, ProblemInstance) else p


def reference_action(p, counters: bool = False, cell_range=None):
    """C restatement of femsched::reference_action (form.hpp:471-595)."""
    cp = _desc(p)
    d = cp.desc
    out = np.zeros(d.output_size, dtype=np.float64)
    cnt = (C.c_longlong * 3)()
    err = C.create_string_buffer(512)
    b, e = cell_range if cell_range else (0, d.cell_count)
    rc = lib().oracle_reference_action_range(C.byref(d), b, e, out.ctypes.data_as(C.POINTER(C.c_double)),
                                             cnt, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return (out, tuple(cnt)) if counters else out


def validate(p):
    cp = _desc(p)
    err = C.create_string_buffer(512)
    rc = lib().oracle_validate(C.byref(cp.desc), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_reference_action(p, counters: bool = False):
    """The reference's own femsched::reference_action, compiled from /root/reference."""
    cp = _desc(p)
    d = cp.desc
    out = np.zeros(d.output_size, dtype=np.float64)
    cnt = (C.c_longlong * 3)()
    err = C.create_string_buffer(512)
    rc = ref().ref_reference_action(C.byref(d), out.ctypes.data_as(C.POINTER(C.c_double)), cnt, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return (out, tuple(cnt)) if counters else out


def ref_time_threads(p, threads: int, reps: int = 1, cell_range=None):
    cp = _desc(p)
    d = cp.desc
    out = np.zeros(d.output_size, dtype=np.float64)
    err = C.create_string_buffer(512)
    b, e = cell_range if cell_range else (0, d.cell_count)
    s = ref().ref_time_threads(C.byref(d), b, e, threads, reps, out.ctypes.data_as(C.POINTER(C.c_double)),
                               err, 512)
    if s < 0:
        raise OracleError(6, err.value.decode())
    return s, out


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def ref_make_problem(op: str, dim: int, degree: int, quad_points: int, cells: int, seed: int) -> ProblemInstance:
    """Instance generated by the reference's own make_problem (preset_map, or generic_map
    with op='generic:<preset>'), converted to the host data model."""
    L = ref()
    err = C.create_string_buffer(512)
    h = L.ref_make_preset(op.encode(), dim, degree, quad_points, cells, seed, err, 512)
    if not h:
        raise OracleError(1, err.value.decode())
    try:
        d = L.ref_instance_desc(h).contents
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
            comps = list(_arr(s.components, s.deriv_terms, np.int32))
            sig.vector_spaces.append(VectorSpace(s.dofs, s.deriv_terms, [int(c) for c in comps]))
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
        p = ProblemInstance(sig, m, tab, conn, sx, vx, d.output_size)
        return p
    finally:
        L.ref_free(h)
