"""GPU action on a renumbered general mesh (femgpu_problem_reorder): the kernels on the reordered
problem, mapped back with the output permutation, match the reference action of the original
(shuffled) problem; and renumbering a shuffled mesh restores the step time of a well-ordered one."""
import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from tests.helpers import max_rel, rel_l2
from tests.test_reorder import shuffled

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fg.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu-marked tests require a B200")


@pytest.mark.parametrize("name,n", [("C2", 6), ("C4", 4), ("C5-hyp-P1", 4), ("C3a", 16)])
def test_reordered_gpu_action_matches_reference_of_the_original(oracle, name, n):
    p = shuffled(name, n)
    q, perms = fg.reorder_problem(p)
    y = fg.output_to_original(fg.gpu_action(q), perms)
    ref = oracle.reference_action(p)
    assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10


def test_reordering_restores_the_step_time():
    p = shuffled("C2", 90)  # maps + x ~ 270 MB: beyond the 126 MB L2
    q, _ = fg.reorder_problem(p)

    def step(prob):
        with fg.GpuInstance(prob) as g:
            g.action()
            g.time_steps(3, pipelined=True)
            return g.time_steps(20, pipelined=True) / 20
    t_shuffled, t_reordered = step(p), step(q)
    assert t_reordered * 2 < t_shuffled, (t_shuffled, t_reordered)
