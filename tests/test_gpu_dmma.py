"""GPU parity of the warp-level FP64 tensor-core family (FEMGPU_DMMA, emit_dmma.cpp).

Same bar as the other families: rel L2 <= 1e-12 (north star) and the reference's elementwise
relative error <= 1e-10 (search.hpp:360-366) against the CPU oracle, over
  * the reference's randomized signatures (test_simulate.cpp:35-56, seed 20240817) with random
    DMMA tilings (cells per tile, T^Q, lanes, warp-task blocking, fragment residency),
  * the acceptance / unit-test tuples (acceptance.cpp:34-37) with partial tiles,
  * every benchmark mesh form at small N, including quadrature tiling (T^Q < Q),
  * the known-answer dense triple product (test_form.cpp:142-193),
  * the non-finite diagnostic (test_form.cpp:270-281)."""
import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import (ACCEPTANCE, DENSE_TRIPLE_PRODUCT_Y, dense_triple_product_problem, max_rel,
                           preset_problem, rel_l2)
from tests.test_gpu_schedules import random_signature

pytestmark = pytest.mark.gpu


def close(y, ref):
    assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10, (rel_l2(y, ref), max_rel(y, ref))


def random_dmma(sig, rng):
    pick = lambda hi: 1 + rng.next_u64() % hi  # noqa: E731
    mb = pick(4)
    joint = [j for j in (1, 2, 3, 4) if mb % j == 0]
    return fg.TilingParams.dmma(cells_per_group=8 * mb, quad_tile=pick(sig.quad_points),
                                lanes_per_cell=(0, 4)[rng.next_u64() % 2], block_cells=32 * pick(8),
                                eval_row_tile=joint[rng.next_u64() % len(joint)],
                                quad_row_tile=rng.next_u64() % 2, stage_smem=rng.next_u64() % 2,
                                basis=abi.BASIS_SMEM if rng.next_u64() % 2 else abi.BASIS_CONST)


def test_dmma_random_signatures(oracle):
    rng = fg.SynthRng(20240817)
    for _ in range(60):
        sig = random_signature(rng)
        cells = 1 + rng.next_u64() % 90
        p = fg.make_problem(sig, fg.generic_map(sig), cells, rng.next_u64())
        ref = oracle.reference_action(p)
        with fg.GpuInstance(p) as g:
            for _ in range(2):
                t = random_dmma(sig, rng)
                close(g.action(t), ref)


@pytest.mark.parametrize("op,d,p,Q", ACCEPTANCE)
def test_dmma_acceptance_tuples(oracle, op, d, p, Q):
    prob = preset_problem(op, d, p, Q, 37, 7)
    ref = oracle.reference_action(prob)
    with fg.GpuInstance(prob) as g:
        close(g.action(fg.TilingParams.dmma()), ref)
        close(g.action(fg.TilingParams.dmma(cells_per_group=16, quad_tile=max(1, Q // 3))), ref)


@pytest.mark.parametrize("form,dim,deg,Q,n", [
    ("laplace", 3, 2, 4, 3), ("helmholtz_coef", 2, 3, 12, 6), ("helmholtz_coef", 3, 3, 24, 2),
    ("elasticity", 3, 2, 4, 3), ("advection", 3, 2, 14, 3), ("advection", 3, 3, 24, 2),
    ("advection", 3, 4, 46, 2), ("hyperelastic", 3, 1, 4, 3), ("hyperelastic", 3, 2, 14, 2),
    ("hyperelastic", 3, 3, 24, 2), ("hyperelastic", 3, 4, 46, 1), ("mass", 2, 1, 3, 9)])
def test_dmma_mesh_forms(oracle, form, dim, deg, Q, n):
    p = fg.mesh_problem(form, dim, deg, Q, n)
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        close(g.action(fg.TilingParams.dmma()), ref)
        close(g.action(fg.TilingParams.dmma(quad_tile=max(1, Q // 4 + 1), cells_per_group=16)), ref)
        close(g.action(fg.TilingParams.dmma(eval_row_tile=2, quad_row_tile=1)), ref)
        close(g.action(fg.TilingParams.dmma(cells_per_group=24, eval_row_tile=3, quad_row_tile=1)), ref)


def test_dmma_known_answer():
    p = dense_triple_product_problem()
    y = fg.gpu_action(p, fg.TilingParams.dmma())
    assert np.max(np.abs(y - DENSE_TRIPLE_PRODUCT_Y) / np.abs(DENSE_TRIPLE_PRODUCT_Y)) <= 1e-13


def test_dmma_nonfinite_names_lowest_cell():
    p = preset_problem("laplace", 2, 2, 6, 40, 7)
    m = p.connectivity.scalar_maps[0].indices
    bad_cells = [23, 31]
    p.scalar_inputs[0][m[bad_cells[0], 0]] = np.nan
    p.scalar_inputs[0][m[bad_cells[1], 0]] = np.inf
    first = int(min(np.nonzero(np.any(np.isin(m, [m[c, 0] for c in bad_cells]), axis=1))[0]))
    with pytest.raises(RuntimeError, match="non-finite value at cell %d during" % first):
        fg.gpu_action(p, fg.TilingParams.dmma())


def test_dmma_infeasible():
    p = preset_problem("mass", 2, 2, 6, 8, 3)
    with pytest.raises(fg.InfeasibleError):
        fg.gpu_action(p, fg.TilingParams.dmma(cells_per_group=12))


def test_dmma_rejects_other_lane_counts():
    p = preset_problem("mass", 2, 2, 6, 8, 3)
    with pytest.raises(fg.InfeasibleError):
        fg.gpu_action(p, fg.TilingParams.dmma(lanes_per_cell=2))
