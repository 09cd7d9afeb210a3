"""Loader for the in-tree libfemgpu.so (the C-ABI of include/femgpu.h).

There is no CPU fallback: if the library is missing every entry point raises
`NativeLibraryMissing`, and on a host without a GPU the device entry points fail
with the CUDA error reported by the library itself.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libfemgpu.so")

EXPORTS = (
    "femgpu_abi_version", "femgpu_last_error", "femgpu_device_count", "femgpu_set_device",
    "femgpu_usable_flops", "femgpu_validate", "femgpu_emit_source", "femgpu_jit_check",
    "femgpu_create", "femgpu_destroy", "femgpu_set_inputs", "femgpu_action", "femgpu_action_host",
    "femgpu_action_device", "femgpu_time_action", "femgpu_execute", "femgpu_default_schedule",
    "femgpu_stats", "femgpu_device_output", "femgpu_stream", "femgpu_action_once",
    "femgpu_host_alloc", "femgpu_host_free", "femgpu_mesh_counts", "femgpu_mesh_build",
    "femgpu_color_cells", "femgpu_profile_action", "femgpu_fp64_peak",
    "femgpu_time_steps", "femgpu_device_input", "femgpu_describe_schedule",
    "femgpu_fp64_dmma_peak", "femgpu_problem_load", "femgpu_problem_free", "femgpu_problem_save",
    "femgpu_schedule_save", "femgpu_schedule_load", "femgpu_action_device_pipelined", "femgpu_check_finite",
    "femgpu_time_steps_ex", "femgpu_reference_counters", "femgpu_read_output", "femgpu_mesh_build_range",
    "femgpu_halo_create", "femgpu_halo_destroy", "femgpu_halo_export", "femgpu_halo_import", "femgpu_halo_action",
    "femgpu_halo_time_steps", "femgpu_halo_check", "femgpu_trace_counters", "femgpu_problem_fuse",
    "femgpu_problem_reorder", "femgpu_action_host_async", "femgpu_action_host_wait",
    "femgpu_cg", "femgpu_halo_cg",
)


class NativeLibraryMissing(RuntimeError):
    pass


class FemgpuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib = None
_lock = threading.Lock()

_P = C.POINTER
_pp = C.POINTER(C.c_void_p)
_dpp = C.POINTER(C.POINTER(C.c_double))


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    "libfemgpu.so is not built (%s); run `make` or __graft_entry__.build()" % LIB_PATH)
            L = C.CDLL(LIB_PATH)
            sig = {
                "femgpu_abi_version": ([], C.c_int32),
                "femgpu_last_error": ([], C.c_char_p),
                "femgpu_device_count": ([], C.c_int32),
                "femgpu_set_device": ([C.c_int32], C.c_int),
                "femgpu_usable_flops": ([_P(abi.Problem), _P(C.c_int64)], C.c_int),
                "femgpu_validate": ([_P(abi.Problem)], C.c_int),
                "femgpu_emit_source": ([_P(abi.Problem), _P(abi.Schedule), C.c_char_p, C.c_size_t,
                                        _P(C.c_size_t)], C.c_int),
                "femgpu_jit_check": ([_P(abi.Problem), _P(abi.Schedule)], C.c_int),
                "femgpu_create": ([_P(abi.Problem), _pp], C.c_int),
                "femgpu_destroy": ([C.c_void_p], C.c_int),
                "femgpu_set_inputs": ([C.c_void_p, _dpp, _dpp], C.c_int),
                "femgpu_action": ([C.c_void_p, _P(abi.Schedule), _P(C.c_double)], C.c_int),
                "femgpu_action_host": ([C.c_void_p, _P(abi.Schedule), _dpp, _dpp, _P(C.c_double)], C.c_int),
                "femgpu_action_host_async": ([C.c_void_p, _P(abi.Schedule), _dpp, _dpp, _P(C.c_double)], C.c_int),
                "femgpu_action_host_wait": ([C.c_void_p], C.c_int),
                "femgpu_cg": ([C.c_void_p, _P(abi.Schedule), C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.c_int32,
                               _P(C.c_int32), _P(C.c_double)], C.c_int),
                "femgpu_action_device": ([C.c_void_p, _P(abi.Schedule), C.c_void_p, C.c_void_p], C.c_int),
                "femgpu_time_action": ([C.c_void_p, _P(abi.Schedule), C.c_int32, C.c_int32, C.c_double,
                                        _P(C.c_double)], C.c_int),
                "femgpu_execute": ([C.c_void_p, _P(abi.Schedule), _P(C.c_double), _P(C.c_double)], C.c_int),
                "femgpu_default_schedule": ([C.c_void_p, _P(abi.Schedule)], C.c_int),
                "femgpu_describe_schedule": ([C.c_void_p, _P(abi.Schedule), C.c_char_p, C.c_size_t,
                                              _P(C.c_size_t)], C.c_int),
                "femgpu_stats": ([C.c_void_p, _P(C.c_int64), _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)], C.c_int),
                "femgpu_device_output": ([C.c_void_p, _P(C.c_void_p)], C.c_int),
                "femgpu_stream": ([C.c_void_p, _P(C.c_void_p)], C.c_int),
                "femgpu_action_once": ([_P(abi.Problem), _P(C.c_double)], C.c_int),
                "femgpu_host_alloc": ([C.c_size_t, _P(C.c_void_p)], C.c_int),
                "femgpu_host_free": ([C.c_void_p], C.c_int),
                "femgpu_mesh_counts": ([C.c_int32, C.c_int32, C.c_int32, _P(C.c_int64), _P(C.c_int64),
                                        _P(C.c_int64), _P(C.c_int32)], C.c_int),
                "femgpu_mesh_build": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P(C.c_int32), _P(C.c_int32),
                                       _P(C.c_double)], C.c_int),
                "femgpu_color_cells": ([_P(C.c_int32), C.c_int32, C.c_int32, C.c_int32, _P(C.c_int32),
                                        _P(C.c_int32)], C.c_int),
                "femgpu_profile_action": ([C.c_void_p, _P(abi.Schedule), C.c_int32, C.c_int32, _P(C.c_double),
                                           _P(C.c_double), _P(C.c_double)], C.c_int),
                "femgpu_fp64_peak": ([_P(C.c_double), _P(C.c_double)], C.c_int),
                "femgpu_fp64_dmma_peak": ([_P(C.c_double)], C.c_int),
                "femgpu_problem_load": ([C.c_char_p, _P(C.c_void_p), _P(_P(abi.Problem))], C.c_int),
                "femgpu_problem_free": ([C.c_void_p], C.c_int),
                "femgpu_problem_fuse": ([_P(_P(abi.Problem)), C.c_int32, _P(C.c_void_p), _P(_P(abi.Problem)),
                                         _P(C.c_int64)], C.c_int),
                "femgpu_problem_reorder": ([_P(abi.Problem), _P(C.c_void_p), _P(_P(abi.Problem)), _P(C.c_int32),
                                            _P(C.c_int32), _P(_P(C.c_int32)), _P(_P(C.c_int32))], C.c_int),
                "femgpu_problem_save": ([_P(abi.Problem), C.c_char_p], C.c_int),
                "femgpu_schedule_save": ([_P(abi.Schedule), C.c_int32, C.c_int32, C.c_char_p], C.c_int),
                "femgpu_schedule_load": ([C.c_char_p, _P(abi.Schedule)], C.c_int),
                "femgpu_time_steps": ([C.c_void_p, _P(abi.Schedule), C.c_int32, _P(C.c_double)], C.c_int),
                "femgpu_time_steps_ex": ([C.c_void_p, _P(abi.Schedule), C.c_int32, C.c_int32, _P(C.c_double)], C.c_int),
                "femgpu_action_device_pipelined": ([C.c_void_p, _P(abi.Schedule), C.c_void_p, C.c_void_p, C.c_void_p],
                                                   C.c_int),
                "femgpu_check_finite": ([C.c_void_p, _P(abi.Schedule), C.c_void_p], C.c_int),
                "femgpu_read_output": ([C.c_void_p, _P(C.c_double)], C.c_int),
                "femgpu_trace_counters": ([C.c_void_p, _P(abi.Schedule), _P(C.c_int64), C.c_int32], C.c_int),
                "femgpu_halo_create": ([C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _P(C.c_int32),
                                        _P(C.c_int32), C.c_int64, _P(C.c_int32), _P(C.c_int32), C.c_int64,
                                        _P(C.c_int32), _P(C.c_int32), _P(C.c_int32), _P(C.c_int32), _pp], C.c_int),
                "femgpu_halo_destroy": ([C.c_void_p], C.c_int),
                "femgpu_halo_export": ([C.c_void_p, C.c_void_p, C.c_size_t, _P(C.c_size_t)], C.c_int),
                "femgpu_halo_import": ([C.c_void_p, C.c_void_p, C.c_size_t], C.c_int),
                "femgpu_halo_action": ([C.c_void_p, _P(abi.Schedule), C.c_void_p, C.c_void_p], C.c_int),
                "femgpu_halo_time_steps": ([C.c_void_p, _P(abi.Schedule), C.c_int32, _P(C.c_double)], C.c_int),
                "femgpu_halo_check": ([C.c_void_p, C.c_void_p], C.c_int),
                "femgpu_halo_cg": ([C.c_void_p, _P(abi.Schedule), C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                                    C.c_int32, _P(C.c_int32), _P(C.c_double)], C.c_int),
                "femgpu_mesh_build_range": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                             _P(C.c_int32), _P(C.c_int32), _P(C.c_double)], C.c_int),
                "femgpu_reference_counters": ([_P(abi.Problem), _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)], C.c_int),
                "femgpu_device_input": ([C.c_void_p, C.c_int32, _P(C.c_void_p)], C.c_int),
            }
            for name, (args, res) in sig.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            if L.femgpu_abi_version() != abi.ABI_VERSION:
                raise NativeLibraryMissing("libfemgpu ABI version mismatch")
            _lib = L
    return _lib


def check(status: int):
    if status != abi.OK:
        raise FemgpuError(status, lib().femgpu_last_error().decode())
