"""Overlapped host-buffer action (csrc/pipeline.cpp): femgpu_action_host uploads x in node-ordered
chunks, runs the action slab by slab over contiguous cell ranges and downloads finished rows of y
while later slabs compute.  It must give the same y as the sequential path and the CPU oracle
(rel L2 <= 1e-12) for every family that supports cell ranges, including changed inputs between calls."""
import ctypes as C

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from paper_2506_17471_b200._native import lib
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu


def pinned(a):
    ptr = C.c_void_p()
    lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
    buf = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
    buf[:] = a
    return buf, ptr


@pytest.mark.parametrize("form,dim,deg,Q,n,scheds", [
    ("laplace", 3, 2, 4, 56, [None, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC), fg.TilingParams.dmma()]),
    ("elasticity", 3, 2, 4, 56, [None, fg.TilingParams.dmma(eval_row_tile=2)]),
    ("mass", 2, 1, 3, 800, [None]),
])
def test_pipelined_host_action_matches_oracle(oracle, monkeypatch, form, dim, deg, Q, n, scheds):
    monkeypatch.setenv("FEMGPU_AUTOTUNE", "0")
    p = fg.mesh_problem(form, dim, deg, Q, n)
    assert p.connectivity.cell_count >= 1000000
    ref = oracle.reference_action(p)
    keep = []
    xs = []
    for x in p.scalar_inputs:
        b, ptr = pinned(x)
        xs.append(b)
        keep.append(ptr)
    vs = []
    for x in p.vector_inputs:
        b, ptr = pinned(x)
        vs.append(b)
        keep.append(ptr)
    yh, ptr = pinned(np.zeros(p.output_size))
    keep.append(ptr)
    with fg.GpuInstance(p) as g:
        for s in scheds:
            yh[:] = np.nan
            g.action_host(xs, vs, yh, s)
            assert g.stats()["launches_last_action"] > 1, "pipelined path not taken"
            assert rel_l2(yh, ref) <= 1e-12, (s, rel_l2(yh, ref))
        # new inputs: the pipeline must upload them (linearity: 2x -> 2y exactly)
        for b in xs + vs:
            b *= 2.0
        g.action_host(xs, vs, yh, scheds[0])
        assert rel_l2(yh, 2.0 * ref) <= 1e-12
        monkeypatch.setenv("FEMGPU_PIPELINE", "0")
        monkeypatch.setenv("FEMGPU_ZERO_OVERLAP", "0")
        y2 = np.array(g.action_host(xs, vs, yh, scheds[0]))
        assert g.stats()["launches_last_action"] == 1
        assert rel_l2(y2, 2.0 * ref) <= 1e-12
    for ptr in keep:
        lib().femgpu_host_free(ptr)


@pytest.mark.parametrize("form,dim,deg,Q,n,sched", [
    ("laplace", 3, 2, 4, 64, None),
    ("laplace", 3, 2, 4, 64, fg.TilingParams.dmma()),
    ("laplace", 3, 2, 4, 64, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC)),
    ("elasticity", 3, 2, 4, 48, fg.TilingParams.dmma()),
    ("helmholtz_coef", 2, 3, 12, 1024, None),
])
@pytest.mark.parametrize("slabs", ["4", "7", "16"])
def test_overlapped_zero_matches_sequential(monkeypatch, form, dim, deg, Q, n, sched, slabs):
    """run_action's fused zeroing (pipeline.cpp overlapped_zero_action): the y rows slab k+2 reaches
    first are cleared by slab k's CTAs, slabs alternate between two streams.  Same
    y as the one-launch path (rel L2 <= 1e-12; the kernels themselves are checked against the oracle
    in test_gpu_parity), also across back-to-back actions, changed inputs and the device path."""
    monkeypatch.setenv("FEMGPU_AUTOTUNE", "0")
    monkeypatch.setenv("FEMGPU_ZERO_SLABS", slabs)
    p = fg.mesh_problem(form, dim, deg, Q, n)
    assert p.output_size >= 1 << 21
    with fg.GpuInstance(p) as g:
        monkeypatch.setenv("FEMGPU_ZERO_OVERLAP", "0")
        ref = np.array(g.action(sched))
        assert g.stats()["launches_last_action"] == 1
        monkeypatch.setenv("FEMGPU_ZERO_OVERLAP", "1")  # the default
        for _ in range(3):
            g.action_device(sched)
        y = np.array(g.action(sched))
        # fewer slabs than requested when a slab would hold less than one wave of CTAs
        assert 4 <= g.stats()["launches_last_action"] <= int(slabs), "fused-zeroing path not taken"
        # every action re-zeroes all of y (a missed chunk would accumulate the previous result)
        assert rel_l2(y, ref) <= 1e-12


FUSED_VARIANTS = {
    "macro-b32": dict(scatter=abi.SCATTER_MACRO, block_cells=32),
    "macro-b32-uncapped": dict(scatter=abi.SCATTER_MACRO, block_cells=32, min_blocks=8),
    "macro-qmajor": dict(scatter=abi.SCATTER_MACRO, block_cells=32, stage_smem=3, reg_target=232),
    "macro-ysmem": dict(scatter=abi.SCATTER_MACRO, stage_smem=2),
    "macro-cp-async": dict(scatter=abi.SCATTER_MACRO, stage_smem=1),
    "scpt-m5": dict(scatter=abi.SCATTER_ATOMIC, block_cells=128, min_blocks=5),
    "scpt-g2": dict(scatter=abi.SCATTER_ATOMIC, group_cells=2),
    "scpt-g2-qloop": dict(scatter=abi.SCATTER_ATOMIC, group_cells=2, stage_smem=4),
    "scpt-g3-qloop-b64": dict(scatter=abi.SCATTER_ATOMIC, group_cells=3, block_cells=64, stage_smem=4),
}


@pytest.mark.parametrize("name", list(FUSED_VARIANTS) + ["dmma", "dmma-joint2", "dmma-prefetch", "dmma-breg"])
def test_fused_zero_every_kernel_variant(monkeypatch, name):
    """Every kernel variant the automatic schedule can pick carries the fused-zeroing prologue:
    three back-to-back fused actions equal the one-launch result (a variant without the prologue
    leaves rows uncleared and accumulates: rel L2 ~ 0.8, 1.6, 2.4, ...)."""
    monkeypatch.setenv("FEMGPU_AUTOTUNE", "0")
    monkeypatch.setenv("FEMGPU_ZERO_SLABS", "7")
    if name.startswith("dmma"):
        knobs = {"dmma": {}, "dmma-joint2": dict(eval_row_tile=2), "dmma-prefetch": dict(quad_row_tile=1, block_cells=256),
                 "dmma-breg": dict(stage_smem=1)}[name]
        s = fg.TilingParams.dmma(**knobs)
    else:
        s = fg.TilingParams.scpt(**FUSED_VARIANTS[name])
    p = fg.mesh_problem("laplace", 3, 2, 4, 64)
    with fg.GpuInstance(p) as g:
        monkeypatch.setenv("FEMGPU_ZERO_OVERLAP", "0")
        ref = np.array(g.action(s))
        monkeypatch.setenv("FEMGPU_ZERO_OVERLAP", "1")
        for i in range(3):
            y = np.array(g.action(s))
            assert g.stats()["launches_last_action"] >= 4, "fused-zeroing path not taken"
            assert rel_l2(y, ref) <= 1e-12, (name, i, rel_l2(y, ref))
