"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle.

Bar: relative L2 <= 1e-12 on y (north star) and the reference's own elementwise
relative error <= 1e-10 (search.hpp:360-366); bitwise equality in strict
(--fmad=false) mode where the summation order is fixed (single cell).
"""
import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import (ACCEPTANCE, DENSE_TRIPLE_PRODUCT_Y, UNIT, dense_triple_product_problem, max_rel,
                           preset_problem, rel_l2)

pytestmark = pytest.mark.gpu

SCHEDULES = {
    "auto": None,
    "scpt-atomic-const": fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, basis=abi.BASIS_CONST),
    "scpt-atomic-smem": fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, basis=abi.BASIS_SMEM),
    "tile-64": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=64),
    "tile-256-smem": fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, block_cells=256, basis=abi.BASIS_SMEM),
    "macro-2": fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=2),
    "macro-4-smem": fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=4, basis=abi.BASIS_SMEM),
}


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fg.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu-marked parity tests require a B200")


def run(g, name, params):
    """Runs a schedule; an explicit macro schedule whose group size does not divide the cell
    count (no common pattern) must be reported infeasible, never silently mis-computed."""
    try:
        return g.action(params)
    except fg.InfeasibleError:
        assert name.startswith("macro") and g.problem.connectivity.cell_count % params.group_cells != 0 \
            or name.startswith("macro") and g.problem.signature.test_dofs >= 1, name
        return None


def check(y, ref, tol_l2=1e-12, tol_el=1e-10):
    if y is None:
        return
    assert y.shape == ref.shape
    assert np.all(np.isfinite(y))
    assert rel_l2(y, ref) <= tol_l2, rel_l2(y, ref)
    assert max_rel(y, ref) <= tol_el, max_rel(y, ref)


@pytest.mark.parametrize("sched", list(SCHEDULES))
@pytest.mark.parametrize("case", ACCEPTANCE, ids=lambda c: "%s-%dd-p%d-q%d" % c)
def test_acceptance_presets(oracle, case, sched):
    p = preset_problem(*case, 16, 7)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        check(run(g, sched, SCHEDULES[sched]), ref)


@pytest.mark.parametrize("case", UNIT, ids=lambda c: "%s-%dd-p%d-q%d-c%d-s%d" % c)
def test_unit_instances(oracle, case):
    p = preset_problem(*case)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for name, s in SCHEDULES.items():
            check(run(g, name, s), ref)


def test_dense_triple_product_known_answer():
    y = fg.gpu_action(dense_triple_product_problem())
    np.testing.assert_allclose(y, DENSE_TRIPLE_PRODUCT_Y, rtol=1e-13, atol=0)


def test_strict_mode_is_bitwise_on_a_single_cell(oracle):
    for op, d, p, Q in ACCEPTANCE:
        prob = preset_problem(op, d, p, Q, 1, 7)
        ref = oracle.reference_action(prob)
        y = fg.gpu_action(prob, fg.TilingParams.scpt(strict=True, scatter=abi.SCATTER_ATOMIC))
        assert np.array_equal(y, ref), (op, d, p, Q, np.max(np.abs(y - ref)))


def test_zero_inputs_give_zero(oracle):
    p = preset_problem("helmholtz", 2, 2, 4, 4, 3)
    p.scalar_inputs = [np.zeros_like(x) for x in p.scalar_inputs]
    assert np.all(fg.gpu_action(p) == 0.0)


def test_linearity_in_trial_dofs():
    p = preset_problem("elasticity", 2, 2, 6, 8, 5)
    base = fg.gpu_action(p)
    q = p.copy()
    q.vector_inputs = [x * 3.7 for x in q.vector_inputs]
    np.testing.assert_allclose(fg.gpu_action(q), 3.7 * base, rtol=1e-12)


def test_non_finite_input_names_cell_and_stage(oracle):
    p = preset_problem("mass", 2, 1, 2, 2, 1)
    p.scalar_inputs[0][0] = np.nan
    with pytest.raises(oracle.OracleError) as ref_err:
        oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for name, s in SCHEDULES.items():
            with pytest.raises(RuntimeError) as e:
                g.action(s)
            if isinstance(e.value, fg.InfeasibleError):
                assert name.startswith("macro"), name
                continue
            assert str(e.value) == str(ref_err.value), name


def test_non_finite_deep_cell_matches_oracle_message(oracle):
    p = preset_problem("laplace", 3, 2, 4, 300, 9)
    p.scalar_inputs[0][p.connectivity.scalar_maps[0].indices[217, 3]] = np.inf
    with pytest.raises(oracle.OracleError) as ref_err:
        oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for name, s in SCHEDULES.items():
            with pytest.raises(RuntimeError) as e:
                g.action(s)
            if isinstance(e.value, fg.InfeasibleError):
                assert name.startswith("macro"), name
                continue
            assert str(e.value) == str(ref_err.value), name


def test_invalid_instance_is_value_error():
    p = preset_problem("mass", 2, 1, 2, 2, 1)
    p.connectivity.test_map.indices[0, 0] = 10 ** 6
    with pytest.raises(ValueError, match="index out of bounds in test space map"):
        fg.gpu_action(p)


MESH_CASES = [("mass", 2, 1, 3, 16), ("laplace", 3, 2, 4, 6), ("helmholtz", 2, 3, 12, 8),
              ("helmholtz_coef", 2, 3, 12, 8), ("helmholtz_coef", 3, 3, 24, 3), ("elasticity", 3, 2, 4, 5),
              ("hyperelasticity", 3, 2, 4, 4), ("advection", 3, 1, 4, 6), ("advection", 3, 2, 14, 4),
              ("hyperelastic", 3, 1, 4, 5), ("hyperelastic", 3, 2, 14, 3)]


@pytest.mark.parametrize("case", MESH_CASES, ids=lambda c: "%s-%dd-p%d-q%d-n%d" % c)
def test_structured_mesh_forms(oracle, case):
    form, d, k, Q, n = case
    p = fg.mesh_problem(form, d, k, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        for name, s in SCHEDULES.items():
            try:
                y = g.action(s)
            except fg.InfeasibleError:
                assert name != "auto"
                continue
            check(y, ref)
        # the default (auto) schedule on these meshes is the macro-element kernel
        assert g.stats()["launches_last_action"] == 1


def test_c1_parity_config_against_reference_build(oracle):
    """C1 (P1 mass, 256x256 unit square) in full against the reference's own build."""
    p = fg.config_problem("C1")
    ref = oracle.ref_reference_action(p) if oracle.ref_available() else oracle.reference_action(p)
    check(fg.gpu_action(p), ref)


def test_executor_outcome(oracle):
    p = preset_problem("laplace", 2, 2, 6, 16, 7)
    ex = fg.gpu_executor()
    out = ex(fg.TilingParams.scpt(), p)
    assert out.ok, out.error
    assert out.measured_seconds is not None and np.isfinite(out.measured_seconds) and out.measured_seconds > 0
    check(out.output, oracle.reference_action(p))


def test_non_affine_instance_matches_oracle(oracle):
    """The reference's non-affine instance (test_io.cpp:10-42, 65-96): coordinates as a vector trial
    space, per-point metric from its derivative terms; no coord map, no affine J."""
    from tests.test_io import non_affine_problem
    p = non_affine_problem()
    ref = oracle.reference_action(p)
    for sched in (None, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC), fg.TilingParams.dmma()):
        y = fg.gpu_action(p, sched)
        assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 4), ("elasticity", 3, 2, 4, 3), ("mass", 2, 1, 3, 12),
                                              ("advection", 3, 2, 14, 3)])
def test_colour_scatter_is_deterministic(oracle, form, dim, deg, Q, n):
    """SCATTER_COLOR: one launch per colour of the test-map colouring, plain y updates: matches the
    oracle and is bitwise identical run to run and across instances."""
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    sched = fg.TilingParams.scpt(scatter=abi.SCATTER_COLOR)
    with fg.GpuInstance(p) as g:
        y1 = g.action(sched)
        y2 = g.action(sched)
        assert g.stats()["launches_last_action"] > 1
    with fg.GpuInstance(p) as g:
        y3 = g.action(sched)
    assert rel_l2(y1, ref) <= 1e-12 and max_rel(y1, ref) <= 1e-10
    assert np.array_equal(y1.view(np.uint64), y2.view(np.uint64))
    assert np.array_equal(y1.view(np.uint64), y3.view(np.uint64))
