"""ctypes mirror of include/femgpu.h (the C-ABI data contract).

Only plain structs and enums live here; the loaders for the product library
(`_native.py`) and for the test oracle (`oracle/oracle.py`) both use these
definitions so that one descriptor feeds both sides of every parity check.
"""
from __future__ import annotations

import ctypes as C

ABI_VERSION = 1

# femgpu_status
OK, E_INVALID, E_INFEASIBLE, E_NONFINITE, E_CUDA, E_JIT, E_INTERNAL = range(7)

# femgpu_map_op == PointwiseMap::Op (form.hpp:194-204) + extension 9
OP_CONSTANT, OP_SCALAR_DERIV, OP_VECTOR_DERIV, OP_JACOBIAN, OP_DETERMINANT, OP_WEIGHT, OP_COORD, \
    OP_ADD, OP_MUL, OP_INV_JACOBIAN = range(10)

SCPT, MLT, DMMA = 0, 1, 2
BASIS_AUTO, BASIS_CONST, BASIS_SMEM = 0, 1, 2
SCATTER_AUTO, SCATTER_ATOMIC, SCATTER_TILE, SCATTER_MACRO, SCATTER_COLOR = 0, 1, 2, 3, 4
FLAG_STRICT, FLAG_FUSED_ZERO, FLAG_PIPE_MEMSET, FLAG_INDEX_LOADS = 1, 2, 4, 8  # femgpu_schedule.reserved[0] flags (femgpu.h)
MAX_SPACES = 8

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class MapNode(C.Structure):
    _fields_ = [("op", C.c_int32), ("a", C.c_int32), ("b", C.c_int32), ("pad_", C.c_int32),
                ("value", C.c_double)]


class Space(C.Structure):
    _fields_ = [("dofs", C.c_int32), ("deriv_terms", C.c_int32), ("components", _ip), ("phi", _dp),
                ("map", _ip), ("global_count", C.c_int32), ("pad_", C.c_int32), ("input", _dp)]


class Problem(C.Structure):
    _fields_ = [
        ("dim", C.c_int32), ("quad_points", C.c_int32), ("coord_dofs", C.c_int32),
        ("affine_geometry", C.c_int32), ("coordinate_space", C.c_int32), ("word_bytes", C.c_int32),
        ("n_scalar", C.c_int32), ("n_vector", C.c_int32),
        ("scalar_spaces", C.POINTER(Space)), ("vector_spaces", C.POINTER(Space)),
        ("test_dofs", C.c_int32), ("test_deriv_terms", C.c_int32),
        ("psi", _dp), ("weights", _dp),
        ("cell_count", C.c_int32), ("test_global_count", C.c_int32),
        ("test_map", _ip), ("coord_map", _ip), ("coords", _dp),
        ("coord_global_count", C.c_int32), ("n_map_nodes", C.c_int32),
        ("map_nodes", C.POINTER(MapNode)), ("map_outputs", _ip),
        ("n_map_outputs", C.c_int32), ("output_size", C.c_int32),
    ]


class Schedule(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("quad_tile", C.c_int32), ("eval_row_tile", C.c_int32),
        ("eval_col_tiles_scalar", C.c_int32 * MAX_SPACES), ("eval_col_tiles_vector", C.c_int32 * MAX_SPACES),
        ("quad_row_tile", C.c_int32), ("quad_col_tile", C.c_int32), ("cells_per_group", C.c_int32),
        ("lanes_per_cell", C.c_int32), ("basis", C.c_int32), ("scatter", C.c_int32),
        ("block_cells", C.c_int32), ("group_cells", C.c_int32), ("reserved", C.c_int32 * 4),
    ]


def dptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def iptr(a):
    return a.ctypes.data_as(_ip) if a is not None else None
