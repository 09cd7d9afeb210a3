"""GPU tests of the paper's schedule space on the sm_100a MLT kernels.

Mirrors the reference's schedule tests (test_simulate.cpp): SCPT and MLT against the oracle,
the plan-structure case, determinism, and the randomized conformance sweep of 220
(signature, tiling) pairs with seed 20240817 over 5-cell instances (:170-203).  Bar: the
reference's elementwise relative error <= 1e-10 (search.hpp:360-366) and rel L2 <= 1e-12."""
import os
import subprocess

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import max_rel, preset_problem, rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def close(y, ref):
    assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10, (rel_l2(y, ref), max_rel(y, ref))


def random_signature(rng):  # test_simulate.cpp:35-56
    pick = lambda hi: 1 + rng.next_u64() % hi  # noqa: E731
    sig = fg.FormSignature(dim=pick(3))
    n_scalar = rng.next_u64() % 3
    n_vector = rng.next_u64() % 2
    for _ in range(n_scalar):
        sig.scalar_spaces.append(fg.ScalarSpace(pick(8), pick(3)))
    for _ in range(n_vector):
        dofs, terms = pick(6), pick(3)
        sig.vector_spaces.append(fg.VectorSpace(dofs, terms, [rng.next_u64() % sig.dim for _ in range(terms)]))
    if not sig.scalar_spaces and not sig.vector_spaces:
        sig.scalar_spaces.append(fg.ScalarSpace(pick(8), pick(3)))
    sig.test_dofs = pick(8)
    sig.test_deriv_terms = pick(3)
    sig.quad_points = pick(9)
    sig.coord_dofs = sig.dim + 1
    return sig


def random_tiling(sig, rng):  # test_simulate.cpp:18-32
    pick = lambda hi: 1 + rng.next_u64() % hi  # noqa: E731
    t = fg.TilingParams(kind=abi.MLT)
    t.quad_tile = pick(sig.quad_points)
    t.eval_row_tile = pick(t.quad_tile)
    t.eval_col_tiles_scalar = [pick(s.dofs) for s in sig.scalar_spaces]
    t.eval_col_tiles_vector = [pick(v.dofs) for v in sig.vector_spaces]
    t.quad_row_tile = pick(sig.test_dofs)
    t.quad_col_tile = pick(t.quad_tile)
    t.cells_per_group = pick(8)
    t.lanes_per_cell = pick(6)
    return t


def test_randomized_conformance_sweep_220(oracle):
    rng = fg.SynthRng(20240817)
    checked = 0
    while checked < 220:
        sig = random_signature(rng)
        p = fg.make_problem(sig, fg.generic_map(sig), 5, rng.next_u64())
        ref = oracle.reference_action(p)
        with fg.GpuInstance(p) as g:
            for _ in range(2):
                t = random_tiling(sig, rng)
                close(g.action(t), ref)
                checked += 1
    assert checked == 220


def test_scpt_and_mlt_match_reference():
    """test_simulate.cpp:60-72, :110-130."""
    from oracle import oracle
    p = preset_problem("laplace", 2, 2, 6, 33, 4)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        close(g.action(fg.TilingParams.scpt()), ref)
        sig = p.signature
        t = fg.TilingParams.untiled(sig, 4, 2)
        t.quad_tile, t.eval_row_tile, t.quad_col_tile = 4, 4, 4
        close(g.action(t), ref)
        close(g.action(fg.TilingParams.untiled(sig, 8, 2)), ref)


def test_mlt_is_repeatable():
    """test_simulate.cpp:132-146 (atomic scatter order may differ; values agree to round-off)."""
    p = preset_problem("mass", 2, 2, 6, 8, 3)
    t = fg.TilingParams.untiled(p.signature, 3, 2)
    with fg.GpuInstance(p) as g:
        a, b = g.action(t), g.action(t)
    assert rel_l2(a, b) <= 1e-15


def test_oversized_workgroup_is_infeasible():
    p = preset_problem("mass", 2, 2, 6, 8, 3)
    t = fg.TilingParams.untiled(p.signature, 64, 32)
    with pytest.raises(fg.InfeasibleError):
        fg.gpu_action(p, t)


def test_mlt_on_high_order_mesh_forms(oracle):
    for args, nc, nwi in [(("helmholtz_coef", 3, 3, 24, 2), 8, 4), (("elasticity", 3, 2, 4, 3), 16, 2),
                          (("hyperelastic", 3, 2, 14, 2), 8, 4)]:
        p = fg.mesh_problem(*args)
        ref = oracle.reference_action(p)
        t = fg.TilingParams.untiled(p.signature, nc, nwi)
        t.quad_tile = max(1, p.signature.quad_points // 2)
        t.eval_row_tile = t.quad_tile
        t.quad_col_tile = t.quad_tile
        close(fg.gpu_action(p, t), ref)


def test_cpp_adapter_drop_in():
    """include/femgpu/femsched_adapter.hpp against the reference's own reference_action and tune
    (binary built in the container from /root/reference headers by tests/cpp/Makefile)."""
    exe = os.path.join(ROOT, "tests", "cpp", "build", "test_adapter")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/build/test_adapter not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


# ---- SCPT with G cells per thread (interleaved statements, shared tabulation loads)
def scpt_g(G, basis=abi.BASIS_AUTO, block=0):
    return fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, group_cells=G, basis=basis, block_cells=block)


def test_scpt_multi_cell_random_signatures(oracle):
    rng = fg.SynthRng(7781)
    for _ in range(40):
        sig = random_signature(rng)
        cells = 1 + rng.next_u64() % 300  # partial last CTA and partial G-slices
        p = fg.make_problem(sig, fg.generic_map(sig), cells, rng.next_u64())
        ref = oracle.reference_action(p)
        with fg.GpuInstance(p) as g:
            G = 2 + rng.next_u64() % 3
            basis = (abi.BASIS_CONST, abi.BASIS_SMEM)[rng.next_u64() % 2]
            close(g.action(scpt_g(G, basis, 32 * (1 + rng.next_u64() % 4))), ref)


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 3), ("advection", 3, 2, 14, 3),
                                              ("helmholtz_coef", 2, 3, 12, 6), ("hyperelastic", 3, 1, 4, 3),
                                              ("elasticity", 3, 2, 4, 2), ("mass", 2, 1, 3, 9)])
def test_scpt_multi_cell_mesh_forms(oracle, form, dim, deg, Q, n):
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for G in (2, 3):
            close(g.action(scpt_g(G)), ref)


def test_scpt_multi_cell_nonfinite_names_lowest_cell():
    p = preset_problem("laplace", 2, 2, 6, 200, 7)
    m = p.connectivity.scalar_maps[0].indices
    bad = [150, 77]
    for c in bad:
        p.scalar_inputs[0][m[c, 0]] = np.nan
    first = int(min(np.nonzero(np.any(np.isin(m, [m[c, 0] for c in bad]), axis=1))[0]))
    with pytest.raises(RuntimeError, match="non-finite value at cell %d during" % first):
        fg.gpu_action(p, scpt_g(3))


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 3), ("mass", 2, 1, 3, 9), ("advection", 3, 1, 4, 3)])
def test_macro_y_accumulators_in_smem(oracle, form, dim, deg, Q, n):
    """Macro family with the y accumulators in thread-private shared memory (stage_smem=2)."""
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        close(g.action(fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, stage_smem=2)), ref)
        close(g.action(fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, stage_smem=2, block_cells=128)), ref)


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 3), ("mass", 2, 1, 3, 9), ("advection", 3, 1, 4, 3),
                                              ("helmholtz_coef", 2, 2, 6, 6)])
def test_macro_quadrature_major(oracle, form, dim, deg, Q, n):
    """Macro family, quadrature-point-major (stage_smem=3): statements interleaved over the group's
    cells so every tabulation load serves all of them."""
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        close(g.action(fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, stage_smem=3)), ref)
        close(g.action(fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, stage_smem=3, block_cells=32, reg_target=232)), ref)


def test_macro_quadrature_major_nonfinite():
    p = fg.mesh_problem("laplace", 3, 2, 4, 3)
    m = p.connectivity.scalar_maps[0].indices
    p.scalar_inputs[0][m[40, 3]] = np.inf
    first = int(np.nonzero(np.any(m == m[40, 3], axis=1))[0].min())
    with pytest.raises(RuntimeError, match="non-finite value at cell %d during" % first):
        fg.gpu_action(p, fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, stage_smem=3))


@pytest.mark.parametrize("form,dim,deg,Q,n", [("helmholtz_coef", 2, 3, 12, 6), ("advection", 3, 2, 14, 2)])
def test_scpt_rolled_quadrature_loop(oracle, form, dim, deg, Q, n):
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for G in (1, 2):
            close(g.action(fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, group_cells=G, stage_smem=4)), ref)


@pytest.mark.parametrize("form,dim,deg,Q,n,G", [("laplace", 3, 2, 4, 4, 6), ("mass", 2, 1, 3, 16, 4), ("advection", 3, 1, 4, 4, 6),
                                                ("helmholtz_coef", 2, 3, 12, 6, 4)])
@pytest.mark.parametrize("stage", [0, 3])
def test_macro_affine_offsets_match_index_loads(oracle, form, dim, deg, Q, n, G, stage):
    """Macro kernels on a lattice-numbered mesh: one index load per map group plus compile-time
    offsets (the default) and the twin that loads every index agree with the reference."""
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for loads in (False, True):
            s = fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=G, stage_smem=stage, index_loads=loads)
            assert ("affine-idx" in g.describe(s)) != loads
            close(g.action(s), ref)


def test_automatic_schedule_keeps_its_index_mode_through_the_python_schedule():
    p = fg.config_problem("C2", n=40)  # 384k cells: timed automatic schedule, macro winner
    with fg.GpuInstance(p) as g:
        y = g.action()
        s = g.default_schedule()
        d = g.describe()
        if d.startswith("femgpu_macro"):
            assert ("affine-idx" in d.split(" | ")[0]) != s.index_loads
        assert rel_l2(g.action(s), y) <= 1e-12
