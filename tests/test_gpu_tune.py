"""GPU tests of the automatic schedule (tune.cpp): the cost model prunes the kernel families, the
survivors are timed once per instance and the winner is cached — the B200 counterpart of the
reference's rank + tune with a measuring Executor (search.hpp:211-416).  Whatever wins, the
action must match the CPU oracle (rel L2 <= 1e-12, elementwise <= 1e-10, search.hpp:360-366)."""
import re

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import max_rel, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("form,dim,deg,Q,n", [("laplace", 3, 2, 4, 33), ("elasticity", 3, 2, 4, 33),
                                              ("helmholtz_coef", 2, 3, 12, 330)])
def test_auto_schedule_is_tuned_and_matches_oracle(oracle, monkeypatch, form, dim, deg, Q, n):
    monkeypatch.setenv("FEMGPU_TUNE_CACHE", "0")
    p = fg.mesh_problem(form, dim, deg, Q, n)
    assert p.connectivity.cell_count >= 200000
    ref = oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        y = g.action()
        assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10
        d = g.describe()
        m = re.search(r"(\d+) compiled, (\d+) timed", d)
        assert "auto:" in d and m, d
        assert int(m.group(2)) <= 10, d  # the paper's b = 9 + SCPT (search.hpp:211-251)
        s = g.default_schedule()
        assert s.kind in (abi.SCPT, abi.DMMA)
        y2 = g.action(s)  # the cached winner, requested explicitly
        assert rel_l2(y2, ref) <= 1e-12
        assert g.describe(s).split(" | ")[0] == d.split(" | ")[0]


def test_small_instances_skip_timing():
    p = fg.mesh_problem("laplace", 3, 2, 4, 4)
    with fg.GpuInstance(p) as g:
        g.action()
        assert "small instance" in g.describe()
        assert g.default_schedule().kind == abi.SCPT


def test_nonfinite_input_survives_tuning(oracle):
    p = fg.mesh_problem("laplace", 3, 2, 4, 33)
    p.scalar_inputs[0][123] = np.nan
    with fg.GpuInstance(p) as g:
        with pytest.raises(RuntimeError, match="non-finite value at cell"):
            g.action()


def test_tuning_decision_is_persisted(tmp_path, monkeypatch):
    monkeypatch.setenv("FEMGPU_CACHE", str(tmp_path))
    monkeypatch.delenv("FEMGPU_TUNE_CACHE", raising=False)
    p = fg.mesh_problem("laplace", 3, 2, 4, 33)
    with fg.GpuInstance(p) as g:
        y1 = g.action()
        assert re.search(r"\d+ timed", g.describe())
        s1 = g.default_schedule()
    assert list(tmp_path.glob("tune_*.txt"))
    with fg.GpuInstance(p) as g:
        y2 = g.action()
        assert "cached decision" in g.describe()
        s2 = g.default_schedule()
    assert (s1.kind, s1.eval_row_tile, s1.quad_tile, s1.block_cells) == (s2.kind, s2.eval_row_tile, s2.quad_tile, s2.block_cells)
    assert rel_l2(y1, y2) <= 1e-12
