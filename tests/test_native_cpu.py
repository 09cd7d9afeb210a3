"""CPU tests of the native library (no GPU): it loads, exports every symbol include/femgpu.h
declares, validates like the reference, emits + NVRTC-compiles sm_100a kernels for every
family, and its mesh generator / colouring are bit-exact against an independent restatement."""
import os
import re

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from oracle import mesh_oracle
from paper_2506_17471_b200 import abi
from paper_2506_17471_b200._native import EXPORTS, LIB_PATH, lib
from tests.golden.make_golden import CASES, key
from tests.helpers import preset_problem
from tests.test_oracle import GOLDEN, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "femgpu.h")).read()
    return sorted(set(re.findall(r"\b(femgpu_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = lib()
    assert L.femgpu_abi_version() == abi.ABI_VERSION
    declared = header_symbols()
    assert declared, "no symbols parsed from include/femgpu.h"
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(EXPORTS)


def test_library_is_sm100a_native():
    out = os.popen("cuobjdump -lelf %s 2>/dev/null" % LIB_PATH).read()
    assert "sm_100a" in out


def test_validation_maps_to_value_error():
    p = preset_problem("mass", 2, 1, 2, 2, 1)
    p.connectivity.scalar_maps[0].indices[1, 0] = -1
    cp = p.to_c()
    import ctypes as C
    assert lib().femgpu_validate(C.byref(cp.desc)) == abi.E_INVALID
    assert b"index out of bounds in scalar space map" in lib().femgpu_last_error()


def test_usable_flops_through_the_abi():
    import ctypes as C
    for op, d, k, q in [("laplace", 2, 2, 6), ("elasticity", 3, 2, 4), ("mass", 3, 1, 5)]:
        p = preset_problem(op, d, k, q, 3, 1)
        v = C.c_int64()
        cp = p.to_c()
        assert lib().femgpu_usable_flops(C.byref(cp.desc), C.byref(v)) == 0
        assert v.value == fg.usable_flops(p.signature)


@pytest.mark.parametrize("sched", ["scpt", "scpt-smem", "macro", "tile"])
@pytest.mark.parametrize("form", [("laplace", 3, 2, 4, 2), ("elasticity", 3, 2, 4, 2), ("helmholtz_coef", 2, 3, 12, 3),
                                  ("advection", 3, 2, 14, 2), ("hyperelastic", 3, 1, 4, 2), ("mass", 2, 1, 3, 4)])
def test_every_kernel_family_compiles_for_sm100a(form, sched):
    p = fg.mesh_problem(*form)
    s = {"scpt": fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC),
         "scpt-smem": fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, basis=abi.BASIS_SMEM),
         "macro": fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=6 if form[1] == 3 else 2),
         "tile": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=64)}[sched]
    src = fg.emit_source(p, s)
    assert "extern \"C\" __global__" in src
    fg.jit_check(p, s)


def test_emitted_map_hoists_cell_invariant_geometry():
    p = fg.mesh_problem("laplace", 3, 2, 4, 2)
    src = fg.emit_source(p, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC))
    body = src.split("femgpu_scpt(")[1].split("femgpu_scpt_checked(")[0]
    hoisted, qloop = body.split("// quadrature point 0", 1)
    # the J^T J metric products are emitted once per cell, before the quadrature points,
    # and no node inside the quadrature points reads the jacobian directly
    import re as _re
    jac_nodes = _re.findall(r"const double (n\d+) = J\d_\d;", hoisted)
    assert len(jac_nodes) >= 9
    assert not _re.search(r"= J\d_\d;", qloop)
    assert body.count("// quadrature point") == 4


@pytest.mark.parametrize("d,n,k,brick", [(2, 3, 1, 2), (2, 4, 3, 8), (3, 2, 2, 1), (3, 3, 2, 2), (3, 2, 4, 4), (3, 5, 1, 4)])
def test_mesh_generator_bitexact(d, n, k, brick):
    node_map, vert_map, coords, n_nodes, n_verts = fg.unit_mesh(d, n, k, brick)
    rn, rv, rc = mesh_oracle.mesh(d, n, k, brick)
    assert np.array_equal(node_map, rn)
    assert np.array_equal(vert_map, rv)
    assert np.array_equal(coords, rc)
    assert n_nodes == (k * n + 1) ** d and n_verts == (n + 1) ** d


def test_mesh_is_conforming_and_positively_oriented():
    node_map, vert_map, coords, n_nodes, _ = fg.unit_mesh(3, 3, 2, 2)
    X = coords[vert_map]
    J = np.stack([X[:, c + 1] - X[:, 0] for c in range(3)], axis=2)
    assert np.all(np.linalg.det(J) > 0)
    assert np.allclose(np.abs(np.linalg.det(J)).sum() / 6.0, 1.0)  # volumes sum to the unit cube
    assert len(np.unique(node_map)) == n_nodes                       # every lattice node is used


def test_colouring_is_valid_and_bitexact():
    node_map, _, _, n_nodes, _ = fg.unit_mesh(3, 3, 2, 2)
    colors, nc = fg.color_cells(node_map, n_nodes)
    assert np.array_equal(colors, mesh_oracle.greedy_colors(node_map))
    assert nc == colors.max() + 1
    for c in range(nc):
        rows = node_map[colors == c].reshape(-1)
        assert len(rows) == len(np.unique(rows))


def test_fails_loudly_without_a_gpu():
    if fg.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        fg.gpu_action(preset_problem("mass", 2, 1, 2, 2, 1))


@pytest.mark.parametrize("case", CASES, ids=key)
def test_reference_counters_through_the_abi_equal_golden(case):
    """femgpu_reference_counters == the ReferenceCounters the reference's own reference_action filled
    (golden vectors written by the reference build, form.hpp:463-472)."""
    p = synth(case)
    assert tuple(fg.reference_counters(p)) == tuple(GOLDEN["counters:" + key(case)])


@pytest.mark.parametrize("stage", [0, 3])
def test_macro_affine_index_pattern(stage):
    """A lattice-numbered structured mesh: every cell group's unique nodes are one base plus fixed
    offsets, so the macro kernels load one index per map group (MacroLayout::aoff);
    FEMGPU_FLAG_INDEX_LOADS and a renumbered mesh fall back to one load per unique node."""
    p = fg.mesh_problem("laplace", 3, 2, 4, 3)
    s = fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=6, stage_smem=stage)
    body = fg.emit_source(p, s).split("_checked(")[0]
    assert "const int igb" in body and body.count("__ldg(&P.gidx") == 2  # node map + coordinate map
    s.index_loads = True
    body = fg.emit_source(p, s).split("_checked(")[0]
    assert "igb" not in body and body.count("__ldg(&P.gidx") > 27
    s.index_loads = False
    rng = np.random.default_rng(3)
    perm = rng.permutation(p.scalar_inputs[0].size).astype(np.int32)
    maps = {id(m): m for m in (p.connectivity.scalar_maps[0], p.connectivity.test_map)}
    for m in maps.values():
        m.indices[:] = perm[m.indices]
    body = fg.emit_source(p, s).split("_checked(")[0]
    assert body.count("const int igb") == 1  # only the (unpermuted) coordinate map stays affine
    fg.jit_check(p, s)
