"""Fused multi-operator actions (csrc/fuse.cpp, femgpu_problem_fuse): the fused
problem's reference action (the CPU oracle, reference_action semantics) is exactly the concatenation
of the separate actions; shared trial spaces and terms are merged; incompatible problems are
rejected (std::invalid_argument -> ValueError, like every invalid instance).  The GPU kernels on
fused problems: tests/test_gpu_fuse.py."""
import numpy as np
import pytest

import paper_2506_17471_b200 as fg


@pytest.mark.parametrize("name", sorted(fg.FUSED_PAIRS))
def test_fused_reference_action_is_the_concatenation(oracle, name):
    a, b = fg.fused_pair(name, n=3)
    f, offs = fg.fuse_problems([a, b])
    assert offs == [0, a.output_size, a.output_size + b.output_size]
    ya, yb = oracle.reference_action(a), oracle.reference_action(b)
    fa, fb = fg.split_output(oracle.reference_action(f), offs)
    # the off-diagonal Psi blocks add exact zeros: bitwise the separate actions
    assert np.array_equal(fa, ya) and np.array_equal(fb, yb)


def test_stokes_pair_shares_the_velocity_space_and_its_divergence_terms():
    a, b = fg.fused_pair("stokes-P2", n=2)
    f, _ = fg.fuse_problems([a, b])
    sig = f.signature
    assert len(sig.vector_spaces) == 1 and sig.vector_spaces[0].deriv_terms == 9  # 9 + 3 terms, 3 shared
    assert not sig.scalar_spaces
    assert sig.test_dofs == a.signature.test_dofs + b.signature.test_dofs
    assert sig.test_deriv_terms == a.signature.test_deriv_terms + b.signature.test_deriv_terms
    psi = f.tabulations.psi
    nWa, Twa = a.signature.test_dofs, a.signature.test_deriv_terms
    assert not psi[:Twa, nWa:].any() and not psi[Twa:, :nWa].any()  # block diagonal


def test_laplace_mass_pair_merges_the_terms_of_one_scalar_space():
    a, b = fg.fused_pair("laplace+mass-P2", n=2)
    f, _ = fg.fuse_problems([a, b])
    assert [s.deriv_terms for s in f.signature.scalar_spaces] == [4]  # 3 gradients + the value
    assert len(f.scalar_inputs) == 1 and np.array_equal(f.scalar_inputs[0], a.scalar_inputs[0])


def test_fusing_three_problems_and_a_problem_with_itself(oracle):
    a, b = fg.fused_pair("laplace+mass-P2", n=2)
    f, offs = fg.fuse_problems([a, b, a])
    assert [s.deriv_terms for s in f.signature.scalar_spaces] == [4]  # a's terms shared with itself
    ys = fg.split_output(oracle.reference_action(f), offs)
    ya = oracle.reference_action(a)
    assert np.array_equal(ys[0], ya) and np.array_equal(ys[2], ya)
    assert np.array_equal(ys[1], oracle.reference_action(b))


def test_different_trial_inputs_stay_separate_spaces(oracle):
    a, b = fg.fused_pair("laplace+mass-P2", n=2)
    b.scalar_inputs = [b.scalar_inputs[0] * 2.0]
    f, offs = fg.fuse_problems([a, b])
    assert len(f.signature.scalar_spaces) == 2
    fa, fb = fg.split_output(oracle.reference_action(f), offs)
    assert np.array_equal(fa, oracle.reference_action(a)) and np.array_equal(fb, oracle.reference_action(b))


def test_incompatible_problems_are_rejected():
    a, b = fg.fused_pair("laplace+mass-P2", n=2)
    w = b.tabulations.weights
    b.tabulations.weights = w * 1.5
    with pytest.raises(ValueError, match="weights"):
        fg.fuse_problems([a, b])
    b.tabulations.weights = w
    c = fg.mesh_problem("mass", 3, 2, 4, 3)  # another mesh size
    with pytest.raises(ValueError, match="differ"):
        fg.fuse_problems([a, c])
    with pytest.raises(ValueError):
        fg.fuse_problems([])


def test_non_affine_problems_fuse_through_their_coordinate_space(oracle):
    """Coordinates as a vector trial space (test_io.cpp:10-42): the fused problem keeps one coordinate
    space (merged), re-pointed by coordinate_space, and reproduces both actions."""
    from tests.test_io import non_affine_problem
    a = non_affine_problem()
    b = non_affine_problem()
    m = b.map  # a second operator: the same DAG with every output doubled
    m.outputs = [m.mul(m.constant(2.0), o) for o in m.outputs]
    f, offs = fg.fuse_problems([a, b])
    assert not f.signature.affine_geometry and len(f.signature.vector_spaces) == 1
    assert f.signature.coordinate_space == 0
    fa, fb = fg.split_output(oracle.reference_action(f), offs)
    assert np.array_equal(fa, oracle.reference_action(a)) and np.array_equal(fb, oracle.reference_action(b))


def test_fusing_a_single_problem_is_the_problem(oracle):
    a, _ = fg.fused_pair("stokes-P2", n=2)
    f, offs = fg.fuse_problems([a])
    assert offs == [0, a.output_size]
    assert np.array_equal(oracle.reference_action(f), oracle.reference_action(a))


def test_fused_then_reordered(oracle):
    """Fusion and renumbering compose: the fused problem of a pair, renumbered, maps back to the two
    separate reference actions."""
    a, b = fg.fused_pair("laplace+mass-P2", n=3)
    f, offs = fg.fuse_problems([a, b])
    q, perms = fg.reorder_problem(f)
    y = fg.output_to_original(oracle.reference_action(q), perms)
    ya, yb = fg.split_output(y, offs)
    from tests.helpers import rel_l2
    assert rel_l2(ya, oracle.reference_action(a)) <= 1e-14 and rel_l2(yb, oracle.reference_action(b)) <= 1e-14


def test_fuse_merges_one_of_two_scalar_spaces(oracle):
    """Helmholtz with a P1 coefficient (two scalar spaces) fused with Laplace on the same P3 field:
    the P3 spaces merge (terms united, the gradients' rows shared when identical), the coefficient
    space stays its own, and both actions are reproduced."""
    a = fg.mesh_problem("helmholtz_coef", 2, 3, 12, 4)
    b = fg.mesh_problem("laplace", 2, 3, 12, 4, seed=11)
    b.tabulations.weights = a.tabulations.weights.copy()
    b.scalar_inputs = [a.scalar_inputs[0].copy()]
    # Laplace's gradient rows equal to Helmholtz's: shared terms
    b.tabulations.scalar_phi = [np.ascontiguousarray(a.tabulations.scalar_phi[0][:2])]
    f, offs = fg.fuse_problems([a, b])
    assert len(f.signature.scalar_spaces) == 2
    assert f.signature.scalar_spaces[0].deriv_terms == a.signature.scalar_spaces[0].deriv_terms
    fa, fb = fg.split_output(oracle.reference_action(f), offs)
    assert np.array_equal(fa, oracle.reference_action(a)) and np.array_equal(fb, oracle.reference_action(b))


def test_c_abi_accepts_null_offsets():
    import ctypes as C
    from paper_2506_17471_b200 import abi
    from paper_2506_17471_b200._native import lib
    a, b = fg.fused_pair("laplace+mass-P2", n=2)
    cps = [a.to_c(), b.to_c()]
    arr = (C.POINTER(abi.Problem) * 2)(*[C.pointer(cp.desc) for cp in cps])
    h = C.c_void_p()
    view = C.POINTER(abi.Problem)()
    assert lib().femgpu_problem_fuse(arr, 2, C.byref(h), C.byref(view), None) == 0
    assert view.contents.output_size == a.output_size + b.output_size
    lib().femgpu_problem_free(h)
