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
        L.ref_save_instance.argtypes = [C.POINTER(abi.Problem), C.c_char_p, C.c_char_p, C.c_int]
        L.ref_load_instance.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.ref_load_instance.restype = C.c_void_p
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
        from paper_2506_17471_b200.io import problem_from_desc
        return problem_from_desc(L.ref_instance_desc(h).contents)
    finally:
        L.ref_free(h)


def ref_save_instance(p, path) -> None:
    """The reference's own femsched::save_instance_file (io.hpp:381-385)."""
    err = C.create_string_buffer(512)
    cp = _desc(p)
    if ref().ref_save_instance(C.byref(cp.desc), str(path).encode(), err, 512):
        raise OracleError(1, err.value.decode())


def ref_load_instance(path) -> ProblemInstance:
    """The reference's own femsched::load_instance_file (io.hpp:387-391)."""
    from paper_2506_17471_b200.io import problem_from_desc
    L = ref()
    err = C.create_string_buffer(512)
    h = L.ref_load_instance(str(path).encode(), err, 512)
    if not h:
        raise OracleError(1, err.value.decode())
    try:
        return problem_from_desc(L.ref_instance_desc(h).contents)
    finally:
        L.ref_free(h)
