"""Locality-restoring renumbering (csrc/reorder.cpp, femgpu_problem_reorder): the reordered
problem's reference action is the original one permuted (up to the order of the per-row sums),
the numbering is first-touch over Morton-sorted cells, square operators keep x and y in one
numbering, and later inputs map through the returned permutations."""
import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from tests.helpers import rel_l2


def shuffled(name, n, seed=3):
    from tools.general_mesh import permuted
    p = fg.config_problem(name, n=n)
    return permuted(p, np.random.default_rng(seed).permutation(p.connectivity.cell_count))


@pytest.mark.parametrize("name,n", [("C2", 4), ("C4", 3), ("C3a", 8), ("C5-adv-P2", 3), ("C5-hyp-P1", 3), ("C1", 16)])
def test_reordered_action_is_the_permuted_action(oracle, name, n):
    p = shuffled(name, n)
    q, perms = fg.reorder_problem(p)
    assert sorted(perms["cells"]) == list(range(p.connectivity.cell_count))
    assert sorted(perms["output"]) == list(range(p.output_size))
    y = fg.output_to_original(oracle.reference_action(q), perms)
    assert rel_l2(y, oracle.reference_action(p)) <= 1e-14


def test_locality_is_restored():
    """After reordering, consecutive cells touch few distinct 64-byte lines of x (8 doubles): a
    64-cell window reads several times fewer lines than in the shuffled numbering."""
    p = shuffled("C2", 12)
    q, _ = fg.reorder_problem(p)

    def lines(prob):
        m = prob.connectivity.scalar_maps[0].indices
        w = m[: (len(m) // 64) * 64].reshape(-1, 64 * m.shape[1]) // 8
        return float(np.mean([len(np.unique(r)) for r in w]))
    assert lines(q) * 3 < lines(p)


def test_square_operator_keeps_one_numbering_and_inputs_map_through():
    p = shuffled("C2", 4)
    q, perms = fg.reorder_problem(p)
    # trial and test spaces share a numbering: output perm == input perm of the scalar space
    assert np.array_equal(perms["output"], perms["scalar"][0])
    assert np.array_equal(q.scalar_inputs[0], p.scalar_inputs[0][perms["scalar"][0]])
    xs, _ = fg.inputs_to_new([p.scalar_inputs[0] * 2.0], [], perms, 3)
    assert np.array_equal(xs[0], q.scalar_inputs[0] * 2.0)


def test_vector_test_space_follows_its_trial_nodes(oracle):
    p = shuffled("C4", 2)
    q, perms = fg.reorder_problem(p)
    node = perms["vector"][0]
    d = 3
    expect = (node[:, None] * d + np.arange(d)[None, :]).reshape(-1)
    assert np.array_equal(perms["output"], expect)
    _, vs = fg.inputs_to_new([], [p.vector_inputs[0]], perms, d)
    assert np.array_equal(vs[0], q.vector_inputs[0])


def test_non_affine_problem_reorders_by_node_index(oracle):
    from tests.test_io import non_affine_problem
    p = non_affine_problem()
    q, perms = fg.reorder_problem(p)
    y = fg.output_to_original(oracle.reference_action(q), perms)
    assert rel_l2(y, oracle.reference_action(p)) <= 1e-14


def test_c_abi_accepts_null_permutation_outputs():
    """femgpu_problem_reorder's permutation outputs are optional (C callers that only want the
    renumbered problem)."""
    import ctypes as C
    from paper_2506_17471_b200 import abi
    from paper_2506_17471_b200._native import lib
    p = shuffled("C2", 3)
    cp = p.to_c()
    h = C.c_void_p()
    view = C.POINTER(abi.Problem)()
    assert lib().femgpu_problem_reorder(C.byref(cp.desc), C.byref(h), C.byref(view), None, None, None, None) == 0
    assert view.contents.cell_count == p.connectivity.cell_count
    lib().femgpu_problem_free(h)
