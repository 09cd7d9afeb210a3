"""The B200 action path behind the reference's operator/plugin seams.

  gpu_action(inst, params=None)      <- femsched::reference_action (form.hpp:471-472): same
                                        signature shape, same exceptions (ValueError for
                                        std::invalid_argument, RuntimeError "non-finite value at
                                        cell N during <stage>", InfeasibleError)
  GpuInstance.action(params)         <- femsched::run_schedule(inst, build_plan(sig, params))
                                        (simulate.hpp:601-603)
  gpu_executor()                     <- femsched::Executor / simulator_executor (search.hpp:257-283):
                                        a callable (TilingParams, ProblemInstance) -> ExecutionOutcome
                                        with measured_seconds from CUDA events

Everything here is a thin ctypes layer over libfemgpu (include/femgpu.h); all
compute runs in the sm_100a kernels the library JIT-compiles.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi
from ._native import FemgpuError, check, lib
from .form import FormSignature, InfeasibleError, ProblemInstance


@dataclass
class TilingParams:
    """femsched::TilingParams (qoi.hpp:23-109) plus B200 knobs (0 = automatic)."""
    kind: int = abi.MLT  # ScheduleKind: abi.SCPT or abi.MLT
    quad_tile: int = 1
    eval_row_tile: int = 1
    eval_col_tiles_scalar: List[int] = field(default_factory=list)
    eval_col_tiles_vector: List[int] = field(default_factory=list)
    quad_row_tile: int = 1
    quad_col_tile: int = 1
    cells_per_group: int = 1
    lanes_per_cell: int = 1
    # B200 knobs
    basis: int = abi.BASIS_AUTO
    scatter: int = abi.SCATTER_AUTO
    block_cells: int = 0
    group_cells: int = 0
    strict: bool = False  # --fmad=false: bitwise per-cell arithmetic of the reference
    reg_target: int = 0
    min_blocks: int = 0
    stage_smem: int = 0  # macro: 1 cp.async staging, 2 y in smem, 3 quadrature-point-major; scpt: 4 rolled q-loop
    split: int = 0  # macro q-major: the G cells of a group split over this many warps (0/1 = one thread per group)
    qmopt: int = 0  # macro q-major: bit 0 hoisted map nodes read back from smem, bit 1 scatter indices reloaded
    fused_zero: bool = False  # y zeroing fused into slab launches (FEMGPU_FLAG_FUSED_ZERO)
    zero_slabs: int = 0  # slabs for fused zeroing (0 = default 8)
    pipe_memset: bool = False  # pipelined actions zero the next output by a memset (FEMGPU_FLAG_PIPE_MEMSET)
    index_loads: bool = False  # macro: load every unique index, no affine offsets (FEMGPU_FLAG_INDEX_LOADS)

    @staticmethod
    def scpt(**knobs) -> "TilingParams":
        return TilingParams(kind=abi.SCPT, **knobs)

    @staticmethod
    def dmma(**knobs) -> "TilingParams":
        """FEMGPU_DMMA: warp-level FP64 tensor-core pipeline (0 = automatic for every field):
        cells_per_group = cells per warp task (8..32, m-blocks of 8), quad_tile = T^Q quadrature
        points per chunk (rounded up to 4: one per lane-group), lanes_per_cell = 4 (fixed by the
        m8n8k4 layout), block_cells = threads per CTA, basis SMEM = fragments staged per CTA."""
        d = dict(kind=abi.DMMA, quad_tile=0, eval_row_tile=0, quad_row_tile=0, quad_col_tile=0,
                 cells_per_group=0, lanes_per_cell=0)
        d.update(knobs)
        return TilingParams(**d)

    @staticmethod
    def untiled(sig: FormSignature, cells_per_group: int = 1, lanes_per_cell: int = 1) -> "TilingParams":
        return TilingParams(kind=abi.MLT, quad_tile=sig.quad_points, eval_row_tile=sig.quad_points,
                            eval_col_tiles_scalar=[s.dofs for s in sig.scalar_spaces],
                            eval_col_tiles_vector=[v.dofs for v in sig.vector_spaces],
                            quad_row_tile=sig.test_dofs, quad_col_tile=sig.quad_points,
                            cells_per_group=cells_per_group, lanes_per_cell=lanes_per_cell)

    def group_size(self) -> int:
        return 32 if self.kind == abi.SCPT else self.cells_per_group * self.lanes_per_cell

    def order_key(self):  # qoi.hpp:95-107
        return [1 if self.kind == abi.SCPT else 0, self.quad_tile, self.eval_row_tile,
                *self.eval_col_tiles_scalar, *self.eval_col_tiles_vector, self.quad_row_tile,
                self.quad_col_tile, self.cells_per_group, self.lanes_per_cell]

    def to_c(self) -> abi.Schedule:
        s = abi.Schedule()
        s.kind = self.kind
        s.quad_tile, s.eval_row_tile = self.quad_tile, self.eval_row_tile
        for i, t in enumerate(self.eval_col_tiles_scalar):
            s.eval_col_tiles_scalar[i] = t
        for i, t in enumerate(self.eval_col_tiles_vector):
            s.eval_col_tiles_vector[i] = t
        s.quad_row_tile, s.quad_col_tile = self.quad_row_tile, self.quad_col_tile
        s.cells_per_group, s.lanes_per_cell = self.cells_per_group, self.lanes_per_cell
        s.basis, s.scatter, s.block_cells = self.basis, self.scatter, self.block_cells
        s.group_cells = self.group_cells
        s.reserved[0] = ((abi.FLAG_STRICT if self.strict else 0) | (abi.FLAG_FUSED_ZERO if self.fused_zero else 0)
                         | (abi.FLAG_PIPE_MEMSET if self.pipe_memset else 0)
                         | (abi.FLAG_INDEX_LOADS if self.index_loads else 0) | (self.zero_slabs & 0xff) << 8)
        s.reserved[1] = self.reg_target
        s.reserved[2] = self.min_blocks
        s.reserved[3] = (self.stage_smem & 0xff) | (self.split & 0xff) << 8 | (self.qmopt & 0xffff) << 16
        return s

    @staticmethod
    def from_c(s: abi.Schedule) -> "TilingParams":
        return TilingParams(kind=s.kind, quad_tile=s.quad_tile, eval_row_tile=s.eval_row_tile,
                            eval_col_tiles_scalar=[t for t in s.eval_col_tiles_scalar if t],
                            eval_col_tiles_vector=[t for t in s.eval_col_tiles_vector if t],
                            quad_row_tile=s.quad_row_tile, quad_col_tile=s.quad_col_tile,
                            cells_per_group=s.cells_per_group, lanes_per_cell=s.lanes_per_cell, basis=s.basis,
                            scatter=s.scatter, block_cells=s.block_cells, group_cells=s.group_cells,
                            strict=bool(s.reserved[0] & abi.FLAG_STRICT), reg_target=s.reserved[1],
                            min_blocks=s.reserved[2], stage_smem=s.reserved[3] & 0xff, split=(s.reserved[3] >> 8) & 0xff,
                            qmopt=(s.reserved[3] >> 16) & 0xffff,
                            fused_zero=bool(s.reserved[0] & abi.FLAG_FUSED_ZERO),
                            zero_slabs=(s.reserved[0] >> 8) & 0xff,
                            pipe_memset=bool(s.reserved[0] & abi.FLAG_PIPE_MEMSET),
                            index_loads=bool(s.reserved[0] & abi.FLAG_INDEX_LOADS))

    def describe(self) -> str:  # search.hpp:301-310
        if self.kind == abi.SCPT:
            return "single-cell-per-work-item"
        tc = "".join("%d," % t for t in self.eval_col_tiles_scalar + self.eval_col_tiles_vector)
        return "mlt(TQ=%d,Ter=%d,Tc=%sTqr=%d,Tqc=%d,Nc=%d,Nwi=%d)" % (
            self.quad_tile, self.eval_row_tile, tc, self.quad_row_tile, self.quad_col_tile,
            self.cells_per_group, self.lanes_per_cell)


def _raise(e: FemgpuError):
    if e.code == abi.E_INVALID:
        raise ValueError(str(e)) from None
    if e.code == abi.E_INFEASIBLE:
        raise InfeasibleError(str(e)) from None
    raise RuntimeError(str(e)) from None


def _call(status: int):
    try:
        check(status)
    except FemgpuError as e:
        _raise(e)


def _sched(params: Optional[TilingParams]):
    if params is None:
        return None
    s = params.to_c()
    return C.byref(s), s


class GpuInstance:
    """A ProblemInstance resident in HBM (femgpu_create), reusable across actions."""

    def __init__(self, problem: ProblemInstance):
        problem.validate()
        self.problem = problem
        self._cp = problem.to_c()
        h = C.c_void_p()
        _call(lib().femgpu_create(C.byref(self._cp.desc), C.byref(h)))
        self._h = h
        self.output_size = problem.output_size

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().femgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def action(self, params: Optional[TilingParams] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        y = out if out is not None else np.empty(self.output_size, dtype=np.float64)
        sp = _sched(params)
        _call(lib().femgpu_action(self._h, sp[0] if sp else None, y.ctypes.data_as(C.POINTER(C.c_double))))
        return y

    def _ptr_array(self, arrays):
        if not arrays:
            return None
        arr = (C.POINTER(C.c_double) * len(arrays))()
        for i, a in enumerate(arrays):
            assert a.dtype == np.float64 and a.flags.c_contiguous
            arr[i] = a.ctypes.data_as(C.POINTER(C.c_double))
        return arr

    def set_inputs(self, scalar_inputs=None, vector_inputs=None):
        _call(lib().femgpu_set_inputs(self._h, self._ptr_array(scalar_inputs), self._ptr_array(vector_inputs)))

    def action_host(self, scalar_inputs, vector_inputs, out: np.ndarray, params: Optional[TilingParams] = None):
        """End to end: H2D of the inputs, the action, D2H of y (femgpu_action_host)."""
        sp = _sched(params)
        _call(lib().femgpu_action_host(self._h, sp[0] if sp else None, self._ptr_array(scalar_inputs),
                                       self._ptr_array(vector_inputs), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def action_host_async(self, scalar_inputs, vector_inputs, out: np.ndarray, params: Optional[TilingParams] = None):
        """Streaming end-to-end step (femgpu_action_host_async): enqueued, completed by
        action_host_wait; the arrays must stay alive and unread until then."""
        sp = _sched(params)
        _call(lib().femgpu_action_host_async(self._h, sp[0] if sp else None, self._ptr_array(scalar_inputs),
                                             self._ptr_array(vector_inputs), out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def action_host_wait(self):
        _call(lib().femgpu_action_host_wait(self._h))

    def action_device(self, params: Optional[TilingParams] = None, y_dev: int = 0, stream: int = 0):
        sp = _sched(params)
        _call(lib().femgpu_action_device(self._h, sp[0] if sp else None, C.c_void_p(y_dev), C.c_void_p(stream)))

    def action_device_pipelined(self, y_dev: int, y_next_dev: int = 0, params: Optional[TilingParams] = None,
                                stream: int = 0):
        """y_dev (all zeros on entry) = A(u) x; y_next_dev zeroed inside the same kernel (stream order)."""
        sp = _sched(params)
        _call(lib().femgpu_action_device_pipelined(self._h, sp[0] if sp else None, C.c_void_p(y_dev),
                                                   C.c_void_p(y_next_dev), C.c_void_p(stream)))

    def check_finite(self, params: Optional[TilingParams] = None, stream: int = 0):
        """Raises RuntimeError('... non-finite value at cell N during <stage>') after device actions."""
        sp = _sched(params)
        _call(lib().femgpu_check_finite(self._h, sp[0] if sp else None, C.c_void_p(stream)))

    def time(self, params: Optional[TilingParams] = None, warmup: int = 5, min_reps: int = 15,
             min_seconds: float = 0.2) -> float:
        """Mean seconds per [zero y + action], paper protocol."""
        s = C.c_double()
        sp = _sched(params)
        _call(lib().femgpu_time_action(self._h, sp[0] if sp else None, warmup, min_reps, min_seconds, C.byref(s)))
        return s.value

    def time_steps(self, steps: int, params: Optional[TilingParams] = None, pipelined: bool = False) -> float:
        """Total seconds of exactly `steps` actions, CUDA events, device sync on both sides.
        pipelined: each step is one femgpu_action_device_pipelined into alternating output buffers
        (one full zeroing + one full action per step, the zeroing inside the action kernel)."""
        s = C.c_double()
        sp = _sched(params)
        _call(lib().femgpu_time_steps_ex(self._h, sp[0] if sp else None, steps, int(pipelined), C.byref(s)))
        return s.value

    def profile(self, params: Optional[TilingParams] = None, warmup: int = 5, reps: int = 50):
        """(step, kernel-only, y-zero) mean seconds, CUDA events on the instance stream."""
        v = [C.c_double() for _ in range(3)]
        sp = _sched(params)
        _call(lib().femgpu_profile_action(self._h, sp[0] if sp else None, warmup, reps, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def default_schedule(self) -> TilingParams:
        """The automatic schedule (femgpu_default_schedule: cost-model pruning + timing, cached)."""
        s = abi.Schedule()
        _call(lib().femgpu_default_schedule(self._h, C.byref(s)))
        return TilingParams.from_c(s)

    def describe(self, params: Optional[TilingParams] = None) -> str:
        """The kernel plan of `params` (None = the automatic schedule with its tuning log)."""
        n = C.c_size_t()
        sp = _sched(params)
        _call(lib().femgpu_describe_schedule(self._h, sp[0] if sp else None, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _call(lib().femgpu_describe_schedule(self._h, sp[0] if sp else None, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def stats(self):
        v = [C.c_int64() for _ in range(4)]
        _call(lib().femgpu_stats(self._h, *[C.byref(x) for x in v]))
        return {"launches_last_action": v[0].value, "device_bytes": v[1].value, "tiles": v[2].value,
                "max_tile_dofs": v[3].value}

    def stream(self) -> int:
        p = C.c_void_p()
        _call(lib().femgpu_stream(self._h, C.byref(p)))
        return p.value or 0

    TRACE_FIELDS = ("barriers_per_workgroup", "flops_matvec", "flops_masked_padding", "gather_words", "scatter_words",
                    "reference_words", "reference_cached_words", "coord_words", "local_eval_read_words",
                    "local_eval_write_words", "local_quad_read_words", "local_words_highwater", "workgroups")

    def trace_counters(self, params: Optional[TilingParams] = None) -> dict:
        """Execution census of the kernel schedule `params` runs (femsched::TraceCounters field names,
        simulate.hpp:91-104, plus ExecutionOutcome::workgroups)."""
        out = (C.c_int64 * len(self.TRACE_FIELDS))()
        sp = _sched(params)
        _call(lib().femgpu_trace_counters(self._h, sp[0] if sp else None, out, len(self.TRACE_FIELDS)))
        return dict(zip(self.TRACE_FIELDS, [int(v) for v in out]))

    def read_output(self) -> np.ndarray:
        """Host copy of the instance's output buffer (the last action's / timed step's y)."""
        y = np.empty(self.problem.output_size, dtype=np.float64)
        _call(lib().femgpu_read_output(self._h, y.ctypes.data_as(C.POINTER(C.c_double))))
        return y

    def device_output(self) -> int:
        p = C.c_void_p()
        _call(lib().femgpu_device_output(self._h, C.byref(p)))
        return p.value or 0


def reference_counters(problem: ProblemInstance):
    """ReferenceCounters of reference_action(p, &c) (form.hpp:463-472): (matvec_mults, matvec_adds,
    map_ops), from the instance's structure (femgpu_reference_counters)."""
    cp = problem.to_c()
    v = [C.c_int64() for _ in range(3)]
    _call(lib().femgpu_reference_counters(C.byref(cp.desc), *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def gpu_action(problem: ProblemInstance, params: Optional[TilingParams] = None, counters: bool = False):
    """reference_action-shaped one-shot: upload, run, download (form.hpp:471-472).  With
    counters=True returns (y, (matvec_mults, matvec_adds, map_ops)) like reference_action with a
    ReferenceCounters argument."""
    with GpuInstance(problem) as g:
        y = g.action(params)
    return (y, reference_counters(problem)) if counters else y


@dataclass
class ExecutionOutcome:
    """femsched::ExecutionOutcome (search.hpp:257-264)."""
    ok: bool = False
    error: str = ""
    output: Optional[np.ndarray] = None
    measured_seconds: Optional[float] = None
    counters: dict = field(default_factory=dict)  # femsched::TraceCounters fields (femgpu_trace_counters)
    workgroups: int = 0


def gpu_executor(measure: bool = True, cache: bool = True):
    """A femsched::Executor-shaped callable backed by the sm_100a kernels (search.hpp:266).
    Instances are uploaded once and cached by identity so tune's candidates share them."""
    instances = {}

    def run(params: TilingParams, inst: ProblemInstance) -> ExecutionOutcome:
        out = ExecutionOutcome()
        try:
            g = instances.get(id(inst)) if cache else None
            if g is None:
                g = GpuInstance(inst)
                if cache:
                    instances[id(inst)] = g
            out.output = g.action(params)
            if measure:
                out.measured_seconds = g.time(params)
            out.counters = g.trace_counters(params)
            out.workgroups = out.counters.pop("workgroups")
            out.ok = True
        except Exception as e:  # search.hpp:278-280: failures become ok=false + message
            out.error = str(e)
        return out

    run.instances = instances
    return run


def emit_source(problem: ProblemInstance, params: Optional[TilingParams] = None) -> str:
    """The CUDA source the JIT compiles for this form (host only; no GPU needed)."""
    cp = problem.to_c()
    n = C.c_size_t()
    sp = _sched(params)
    _call(lib().femgpu_emit_source(C.byref(cp.desc), sp[0] if sp else None, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _call(lib().femgpu_emit_source(C.byref(cp.desc), sp[0] if sp else None, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def jit_check(problem: ProblemInstance, params: Optional[TilingParams] = None) -> None:
    """NVRTC-compiles the emitted kernel for sm_100a (host only)."""
    cp = problem.to_c()
    sp = _sched(params)
    _call(lib().femgpu_jit_check(C.byref(cp.desc), sp[0] if sp else None))


def fp64_peaks():
    """Live FP64 peaks of the current device: {"dfma": TF, "dmma": TF, "fp64": max, "sm_ghz": nominal}."""
    t, g, m = C.c_double(), C.c_double(), C.c_double()
    _call(lib().femgpu_fp64_peak(C.byref(t), C.byref(g)))
    _call(lib().femgpu_fp64_dmma_peak(C.byref(m)))
    return {"dfma": t.value, "dmma": m.value, "fp64": max(t.value, m.value), "sm_ghz": g.value}


def fp64_peak():
    """(TFLOP/s, nominal SM GHz): live DFMA peak of the current device (femgpu_fp64_peak)."""
    t, g = C.c_double(), C.c_double()
    _call(lib().femgpu_fp64_peak(C.byref(t), C.byref(g)))
    return t.value, g.value


def device_count() -> int:
    return int(lib().femgpu_device_count())
