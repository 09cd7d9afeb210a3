"""CPU tests: the oracle (C restatement of femsched::reference_action) pinned against the
reference's own code (oracle/_ref) and the committed golden vectors, plus the reference's own
known-answer and property tests restated (test_form.cpp)."""
import hashlib
import os

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from tests.golden.make_golden import CASES, instance_digest, key
from tests.helpers import (ACCEPTANCE, DENSE_TRIPLE_PRODUCT_Y, dense_triple_product_problem, max_rel,
                           preset_problem, rel_l2)

GOLDEN = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.npz"))


def synth(case):
    op, d, p, q, cells, seed = case
    if op.startswith("generic:"):
        sig = fg.preset_signature(op[8:], d, p, q)
        return fg.synthesize_problem(sig, cells, seed)
    return preset_problem(op, d, p, q, cells, seed)


@pytest.mark.parametrize("case", CASES, ids=key)
def test_synthesis_matches_reference_make_problem(case):
    """The numpy make_problem draws the same splitmix64 stream as form.hpp:774-852."""
    p = synth(case)
    digest = bytes(GOLDEN["digest:" + key(case)]).decode()
    assert instance_digest(p) == digest


@pytest.mark.parametrize("case", CASES, ids=key)
def test_oracle_bitwise_equals_reference_golden(oracle, case):
    p = synth(case)
    y, cnt = oracle.reference_action(p, counters=True)
    assert np.array_equal(y, GOLDEN["y:" + key(case)])
    assert tuple(cnt) == tuple(GOLDEN["counters:" + key(case)])


def test_oracle_bitwise_equals_reference_build_on_meshes(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent on this host)")
    for args in [("laplace", 3, 2, 4, 3), ("helmholtz_coef", 2, 3, 12, 5), ("elasticity", 3, 2, 4, 2),
                 ("advection", 3, 2, 14, 2), ("hyperelastic", 3, 2, 14, 2), ("mass", 2, 1, 3, 8)]:
        p = fg.mesh_problem(*args)
        assert np.array_equal(oracle.reference_action(p), oracle.ref_reference_action(p)), args


def test_dense_triple_product_known_answer(oracle):
    """test_form.cpp:142-193."""
    y = oracle.reference_action(dense_triple_product_problem())
    assert np.array_equal(y, DENSE_TRIPLE_PRODUCT_Y)
    # the hand check: y0 = det * sum_i (0.3+0.1 i) w_i u_i, u_i = 4.4 + i
    u = np.array([4.4 + i for i in range(5)])
    assert abs(y[0] - 3.0 * np.sum((0.3 + 0.1 * np.arange(5)) * np.array([0.5, 0.6, 0.7, 0.8, 0.9]) * u)) < 1e-12


def test_zero_in_zero_out(oracle):
    p = preset_problem("helmholtz", 2, 2, 4, 4, 3)
    p.scalar_inputs = [np.zeros_like(x) for x in p.scalar_inputs]
    assert np.all(oracle.reference_action(p) == 0.0)


def test_shared_dofs_sum_cell_contributions(oracle):
    """test_form.cpp:195-204."""
    p = preset_problem("laplace", 2, 2, 6, 2, 11)
    whole = oracle.reference_action(p)
    first = oracle.reference_action(p, cell_range=(0, 1))
    second = oracle.reference_action(p, cell_range=(1, 2))
    np.testing.assert_allclose(whole, first + second, rtol=0, atol=1e-14)


def test_linearity(oracle):
    """test_form.cpp:206-217."""
    p = preset_problem("elasticity", 2, 2, 6, 8, 5)
    base = oracle.reference_action(p)
    q = p.copy()
    q.vector_inputs = [x * 3.7 for x in q.vector_inputs]
    np.testing.assert_allclose(oracle.reference_action(q), 3.7 * base, rtol=1e-12)


def test_cell_order_only_reassociates(oracle):
    """test_form.cpp:219-241."""
    p = preset_problem("helmholtz", 2, 1, 3, 10, 13)
    base = oracle.reference_action(p)
    r = p.copy()
    for m in r.connectivity.scalar_maps + [r.connectivity.test_map, r.connectivity.coord_map]:
        m.indices = m.indices[::-1].copy()
    assert max_rel(oracle.reference_action(r), base) <= 1e-10


def test_counters_equal_usable_flops(oracle):
    """test_form.cpp:243-252."""
    sig = fg.preset_signature("laplace", 2, 2, 6)
    p = fg.make_problem(sig, fg.preset_map("laplace", sig), 3, 2)
    _, (mults, adds, mapops) = oracle.reference_action(p, counters=True)
    assert mults == 3 * fg.usable_flops(sig) // 2 and adds == 3 * fg.usable_flops(sig) // 2 and mapops > 0


def test_usable_flops_and_presets():
    """test_form.cpp:28-107."""
    assert fg.usable_flops(fg.preset_signature("laplace", 2, 2, 6)) == 288
    m = fg.FormSignature(dim=1, scalar_spaces=[fg.ScalarSpace(1, 1)], test_dofs=1, test_deriv_terms=1,
                         quad_points=1, coord_dofs=2)
    assert fg.usable_flops(m) == 4
    e = fg.preset_signature("elasticity", 3, 2, 10)
    assert (e.vector_spaces[0].dofs, e.vector_spaces[0].deriv_terms, e.test_dofs, e.test_deriv_terms) == (10, 9, 30, 9)
    assert fg.simplex_space_dim(2, 2) == 6 and fg.simplex_space_dim(3, 3) == 20 and fg.simplex_space_dim(0, 3) == 1
    for bad in [("elasticity", 1, 2, 4), ("mass", 2, 0, 4), ("mass", 2, 2, 0)]:
        with pytest.raises(ValueError):
            fg.preset_signature(*bad)


def test_non_finite_diagnostic_names_cell_and_stage(oracle):
    """test_form.cpp:270-281, and the same message as the compiled reference."""
    p = preset_problem("mass", 2, 1, 2, 2, 1)
    p.scalar_inputs[0][0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.reference_action(p)
    assert "cell 0" in str(e.value) and "evaluation" in str(e.value)
    if oracle.ref_available():
        with pytest.raises(oracle.OracleError) as r:
            oracle.ref_reference_action(p)
        assert str(r.value) == str(e.value)


def test_validation_messages_match_reference(oracle):
    p = preset_problem("mass", 2, 1, 2, 2, 1)
    p.connectivity.test_map.indices[0, 0] = 10 ** 6
    with pytest.raises(oracle.OracleError, match="index out of bounds in test space map"):
        oracle.reference_action(p)
    if oracle.ref_available():
        with pytest.raises(oracle.OracleError, match="index out of bounds in test space map"):
            oracle.ref_reference_action(p)


def test_acceptance_tuples_against_reference_build(oracle):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    for op, d, p_, q in ACCEPTANCE:
        ref = oracle.ref_make_problem(op, d, p_, q, 16, 7)
        assert np.array_equal(oracle.reference_action(ref), oracle.ref_reference_action(ref))
        assert rel_l2(oracle.reference_action(synth((op, d, p_, q, 16, 7))), oracle.ref_reference_action(ref)) == 0.0
