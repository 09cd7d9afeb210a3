"""GPU parity at the benchmark sizes: every SURVEY §8d configuration at its configured N with the
automatic schedule, against the reference's own reference_action (oracle/_ref, all host threads;
the C restatement on a cell sample where the reference build is absent).  The bar is the
reference's tune check (elementwise relative error <= 1e-10, search.hpp:360-366) and the north
star's relative L2 <= 1e-12.  Also: the output-pipelined action (the bench step), a
reference-written instance file run through the kernels (io.hpp:381-391), the device-side
non-finite check and the host pipeline on a test numbering with a gap of untouched rows."""
import os

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi
from tests.helpers import complete_rows, max_rel, rel_l2

pytestmark = pytest.mark.gpu
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")
THREADS = max(1, min(os.cpu_count() or 1, 64))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fg.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu-marked tests require a B200")


def reference(oracle, p):
    """(reference y, rows to compare): the full reference action, or (no reference build on this
    host) the C restatement over a cell sample and the rows it completes."""
    if oracle.ref_available():
        _, ref = oracle.ref_time_threads(p, THREADS, reps=1)
        return ref, None
    m = min(p.connectivity.cell_count, 50000)
    return oracle.reference_action(p, cell_range=(0, m)), complete_rows(p, m)


@pytest.mark.parametrize("name", list(fg.CONFIGS))
def test_benchmark_config_at_full_size_matches_reference(oracle, name):
    p = fg.config_problem(name)
    with fg.GpuInstance(p) as g:
        y = g.action()  # the automatic schedule
        g.time_steps(3, pipelined=True)  # the bench step: output-pipelined actions
        yp = g.read_output()
    ref, rows = reference(oracle, p)
    for out in (y, yp):
        a, b = (out, ref) if rows is None else (out[rows], ref[rows])
        assert np.all(np.isfinite(a))
        assert rel_l2(a, b) <= 1e-12, (name, rel_l2(a, b))
        assert max_rel(a, b) <= 1e-10, (name, max_rel(a, b))


@pytest.mark.parametrize("sched", [None, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC),
                                   fg.TilingParams.dmma(), fg.TilingParams.untiled(
                                       fg.preset_signature("laplace", 3, 2, 4), 32, 1)],
                         ids=["auto", "scpt", "dmma", "mlt"])
def test_pipelined_action_alternating_outputs(oracle, sched):
    """femgpu_action_device_pipelined: y (zeroed on entry) = A x and the next output zeroed in the
    same launch; chained over alternating buffers every step equals the reference."""
    import torch
    p = fg.config_problem("C2", n=12)
    ref = oracle.reference_action(p)
    n = p.output_size
    with fg.GpuInstance(p) as g:
        bufs = [torch.zeros(n, dtype=torch.float64, device="cuda"),
                torch.full((n,), 7.0, dtype=torch.float64, device="cuda")]  # garbage: must be zeroed
        stream = torch.cuda.current_stream().cuda_stream or 1
        for k in range(4):
            g.action_device_pipelined(bufs[k & 1].data_ptr(), bufs[(k + 1) & 1].data_ptr(), sched, stream=stream)
            torch.cuda.synchronize()
            y = bufs[k & 1].cpu().numpy()
            assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10, k
            assert not bufs[(k + 1) & 1].any().item(), "next output not zeroed"


@pytest.mark.parametrize("fname,key,npz", [
    ("instance_laplace_2d_p2.txt", "y:laplace|2|2|6|16|7", "reference_outputs.npz"),
    ("mesh_helmholtz_coef_2d_p3.txt", "y:mesh_helmholtz_coef_2d_p3", "mesh_instance_outputs.npz"),
    ("mesh_elasticity_3d_p2.txt", "y:mesh_elasticity_3d_p2", "mesh_instance_outputs.npz")])
def test_reference_written_instance_file_through_the_kernels(fname, key, npz):
    """Instance files written by the reference's own femsched::save_instance_file (io.hpp:381-385)
    load through femgpu_problem_load and run through the kernels to the y the reference's
    reference_action produced for them (tests/golden/make_golden.py)."""
    p = fg.load_instance(os.path.join(GOLDEN_DIR, fname))
    ref = np.load(os.path.join(GOLDEN_DIR, npz))[key]
    for sched in (None, fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC), fg.TilingParams.dmma()):
        y = fg.gpu_action(p, sched)
        assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10, (fname, sched)


def test_device_action_reports_non_finite_on_request(oracle):
    """femgpu_action_device has no host sync; femgpu_check_finite afterwards reports the
    reference's diagnostic (form.hpp:492-595) for a NaN input."""
    import torch
    p = fg.config_problem("C2", n=6)
    bad = 123
    p.scalar_inputs[0][p.connectivity.scalar_maps[0].indices[bad, 0]] = np.nan
    with pytest.raises(RuntimeError) as ref_err:
        oracle.ref_reference_action(p) if oracle.ref_available() else oracle.reference_action(p)
    with fg.GpuInstance(p) as g:
        y = torch.zeros(p.output_size, dtype=torch.float64, device="cuda")
        g.action_device(y_dev=y.data_ptr())
        with pytest.raises(RuntimeError) as err:
            g.check_finite()
    assert str(err.value) == str(ref_err.value)


def test_host_pipeline_with_a_gap_of_untouched_rows(oracle):
    """femgpu_action_host's overlapped download must not copy rows before they are
    zeroed when the test numbering leaves a block of rows no cell touches."""
    p = fg.config_problem("C2", n=56)  # > 1M cells: the overlapped host pipeline applies
    tm = p.connectivity.test_map
    gap, mid = 1 << 20, tm.global_count // 2
    idx = tm.indices.astype(np.int64)
    idx[idx >= mid] += gap
    p.connectivity.test_map = fg.IndexMap(idx.astype(np.int32), tm.global_count + gap)
    p.output_size = tm.global_count + gap
    p.validate()
    ref = oracle.reference_action(p)
    assert not ref[mid:mid + gap].any()
    with fg.GpuInstance(p) as g:
        for _ in range(2):  # the second call runs on a dirty output buffer
            yh = np.full(p.output_size, np.nan)
            g.action_host(list(p.scalar_inputs), list(p.vector_inputs), yh)
            assert rel_l2(yh, ref) <= 1e-12 and max_rel(yh, ref) <= 1e-10


def test_executor_fills_trace_counters():
    """ExecutionOutcome::counters (search.hpp:257-264) from femgpu_trace_counters: the usable matvec
    flops are exact; the macro layout reads each unique node of a group once, so it gathers and
    scatters fewer words than one-thread-per-cell SCPT; DMMA reports its m8n8k4 padding."""
    p = fg.config_problem("C2", n=10)
    run = fg.gpu_executor(measure=False)
    cells, usable = p.connectivity.cell_count, fg.usable_flops(p.signature)
    scpt = run(fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC), p)
    macro = run(fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=6, block_cells=32), p)
    dmma = run(fg.TilingParams.dmma(), p)
    for o in (scpt, macro, dmma):
        assert o.ok and o.counters["flops_matvec"] == usable * cells and o.workgroups > 0
    assert scpt.counters["gather_words"] == 10 * cells and scpt.counters["scatter_words"] == 10 * cells
    assert macro.counters["gather_words"] == 27 * cells // 6 and macro.counters["scatter_words"] == 27 * cells // 6
    assert macro.counters["coord_words"] == 3 * 8 * cells // 6 and scpt.counters["coord_words"] == 3 * 4 * cells
    assert dmma.counters["flops_masked_padding"] > 0 and scpt.counters["flops_masked_padding"] == 0
