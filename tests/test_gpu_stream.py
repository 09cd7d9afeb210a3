"""Streaming end-to-end actions (femgpu_action_host_async / _wait): two device buffer sets alternate
so consecutive steps overlap their uploads and downloads.  Every step's output equals the reference
action of that step's inputs; the instance ends holding the last step; a non-finite value in any
step is reported by the wait; other calls complete pending steps first."""
import ctypes as C

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200._native import lib
from tests.helpers import max_rel, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fg.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu-marked tests require a B200")


class Pinned:
    def __init__(self):
        self.ptrs = []

    def like(self, a):
        ptr = C.c_void_p()
        lib().femgpu_host_alloc(a.nbytes, C.byref(ptr))
        buf = np.ctypeslib.as_array((C.c_double * a.size).from_address(ptr.value))
        buf[:] = a
        self.ptrs.append(ptr)
        return buf

    def free(self):
        for p in self.ptrs:
            lib().femgpu_host_free(p)


@pytest.mark.parametrize("name,n", [("C2", 60), ("C4", 56)])  # >= 1M cells: the slab pipeline applies
def test_streaming_steps_match_the_reference_per_step(oracle, name, n):
    p = fg.config_problem(name, n=n)
    pin = Pinned()
    steps = 5
    try:
        xs = [[pin.like(x * (1.0 + 0.1 * k)) for x in p.scalar_inputs] for k in range(steps)]
        vs = [[pin.like(v * (1.0 + 0.1 * k)) for v in p.vector_inputs] for k in range(steps)]
        ys = [pin.like(np.zeros(p.output_size)) for _ in range(steps)]
        with fg.GpuInstance(p) as g:
            g.action()
            for k in range(steps):
                g.action_host_async(xs[k], vs[k], ys[k])
            g.action_host_wait()
            last = g.read_output()
        m = min(p.connectivity.cell_count, 100000)
        from tests.helpers import complete_rows
        rows = complete_rows(p, m)
        for k in range(steps):
            p.scalar_inputs = [np.array(x) for x in xs[k]]
            p.vector_inputs = [np.array(v) for v in vs[k]]
            ref = oracle.reference_action(p, cell_range=(0, m))
            y = np.array(ys[k])
            assert rel_l2(y[rows], ref[rows]) <= 1e-12 and max_rel(y[rows], ref[rows]) <= 1e-10, k
        assert np.array_equal(last, np.array(ys[-1]))
    finally:
        pin.free()


def test_streaming_non_finite_is_reported_by_the_wait():
    p = fg.config_problem("C2", n=60)
    pin = Pinned()
    try:
        good = [pin.like(x) for x in p.scalar_inputs]
        bad = [pin.like(x) for x in p.scalar_inputs]
        bad[0][17] = np.nan
        y0, y1 = pin.like(np.zeros(p.output_size)), pin.like(np.zeros(p.output_size))
        with fg.GpuInstance(p) as g:
            g.action()
            g.action_host_async(good, [], y0)
            g.action_host_async(bad, [], y1)
            with pytest.raises(RuntimeError, match="non-finite value at cell"):
                g.action_host_wait()
            # the instance recovers: a synchronous action on good inputs
            g.set_inputs([np.array(x) for x in good], [])
            assert np.all(np.isfinite(g.action()))
    finally:
        pin.free()


def test_other_calls_complete_pending_steps_first():
    """A synchronous action, a schedule change and set_inputs each drain the pending steps; after an
    even number of steps (the last one in buffer set 1) the instance holds that step's inputs."""
    p = fg.config_problem("C2", n=60)
    pin = Pinned()
    try:
        xs = [[pin.like(x * (1.0 + 0.25 * k)) for x in p.scalar_inputs] for k in range(4)]
        ys = [pin.like(np.zeros(p.output_size)) for _ in range(4)]
        with fg.GpuInstance(p) as g:
            want = []
            for k in range(4):
                g.set_inputs([np.array(x) for x in xs[k]], [])
                want.append(g.action())
            g.action_host_async(xs[0], [], ys[0])
            g.action_host_async(xs[1], [], ys[1])
            y_sync = g.action()  # drains: the instance now holds step 1's inputs (set 1 copied back)
            assert rel_l2(y_sync, want[1]) <= 1e-12
            g.action_host_async(xs[2], [], ys[2])
            g.action_host_async(xs[3], [], ys[3], params=fg.TilingParams.scpt())  # another schedule: drains first
            g.action_host_wait()
            for k in range(4):
                y = np.array(ys[k])
                assert rel_l2(y, want[k]) <= 1e-12 and max_rel(y, want[k]) <= 1e-10, k
            assert rel_l2(g.read_output(), want[3]) <= 1e-12
            g.action_host_async(xs[0], [], ys[0])
            g.set_inputs([np.array(x) for x in xs[2]], [])  # drains, then replaces the inputs
            assert rel_l2(np.array(ys[0]), want[0]) <= 1e-12
            assert rel_l2(g.action(), want[2]) <= 1e-12
    finally:
        pin.free()
