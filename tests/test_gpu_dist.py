"""GPU tests of the cell-partitioned action with the GPU-to-GPU exchange (csrc/halo.cu).

The box has one GPU, so ranks share cuda:0:
* in one process, one thread per rank (peer pointers used directly, kernels of the ranks run
  concurrently): world 2 and 3, scalar / vector / coefficient forms, inputs changing between
  actions (ghost inputs poisoned with NaN on the device: the pull must refill them), and a
  distributed CG through DistOperator;
* two processes launched by bench.py --gpus 2 itself (CUDA IPC path, the multi-GPU bench leg):
  parity of the gathered owned rows against the reference CPU action."""
import ctypes as C
import json
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import dist as fdist
from tests.helpers import max_rel, rel_l2
from tests.test_dist import ThreadGather

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if fg.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu-marked tests require a B200")


def run_ranks(world, fn):
    """fn(rank, gather) in `world` threads; re-raises the first failure."""
    tg = ThreadGather(world)
    res, err = [None] * world, []

    def body(r):
        try:
            from paper_2506_17471_b200._native import lib
            lib().femgpu_set_device(0)
            res[r] = fn(r, tg.for_rank(r))
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            tg.bar.abort()
    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return res


def device_view(inst, space, n, comps, stride):
    import torch
    from paper_2506_17471_b200.krylov import _CudaArray
    from paper_2506_17471_b200._native import lib
    p = C.c_void_p()
    lib().femgpu_device_input(inst.handle, space, C.byref(p))
    t = torch.as_tensor(_CudaArray(p.value, n * stride), device="cuda")
    return t.view(n, stride)[:, :comps]


FORMS = [("laplace", 3, 2, 4, 6), ("elasticity", 3, 2, 4, 4), ("helmholtz_coef", 2, 3, 12, 12),
         ("hyperelastic", 3, 2, 14, 2)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("args", FORMS, ids=lambda a: "-".join(map(str, a)))
def test_halo_action_matches_oracle_with_changing_inputs(oracle, args, world):
    import torch
    p = fg.mesh_problem(*args)
    d = p.signature.dim
    ns = len(p.scalar_inputs)

    def new_x(gl, comps, step):
        return (0.5 + 0.25 * step + 1e-3 * ((gl[:, None] * comps + np.arange(comps)) % 97))

    def rank(r, gather):
        plan = fdist.build_plan(fdist.rank_slab(args, r, world), r, world, gather)
        di = fdist.DistInstance(plan, gather)
        out = []
        try:
            for step in range(3):
                if step:  # new owned inputs uploaded on the instance stream, ghosts poisoned (NaN)
                    xs = []
                    for s, gl in enumerate(plan.trial_global):
                        comps = 1 if s < ns else d
                        v = new_x(gl, comps, step)
                        for q, (mine, _) in plan.pull[s].items():
                            v[mine] = np.nan
                        xs.append(np.ascontiguousarray(v.reshape(-1)))
                    # (femgpu_set_inputs: stream-ordered copies only -- a device-wide synchronising
                    # call would wait for the other ranks' exchange kernels, which wait for this rank)
                    di.inst.set_inputs(xs[:ns], xs[ns:])
                di.action()
                di.check()
                out.append(di.owned_output())
        finally:
            di.close()
        return out

    res = run_ranks(world, rank)
    for step in range(3):
        if step:
            for i in range(ns):
                g = np.arange(len(p.scalar_inputs[i]))
                p.scalar_inputs[i] = new_x(g, 1, step).reshape(-1)
            for i in range(len(p.vector_inputs)):
                g = np.arange(len(p.vector_inputs[i]) // d)
                p.vector_inputs[i] = new_x(g, d, step).reshape(-1)
        ref = oracle.reference_action(p)
        y = np.full(p.output_size, np.nan)
        for r in range(world):
            g, v = res[r][step]
            assert np.all(np.isnan(y[g]))
            y[g] = v
        assert not np.isnan(y).any(), step
        assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10, (step, rel_l2(y, ref))


def test_distributed_device_cg(oracle):
    """dist_cg with the distributed action on the device (DistOperator): the assembled solution
    satisfies the global A x = b of the oracle."""
    import torch
    args = ("helmholtz", 3, 2, 14, 4)
    world = 2

    def rank(r, gather):
        slab = fdist.rank_slab(args, r, world)
        tab = slab.local.tabulations
        tab.psi = np.ascontiguousarray(np.transpose(tab.scalar_phi[0], (0, 2, 1)))
        plan = fdist.build_plan(slab, r, world, gather)
        di = fdist.DistInstance(plan, gather)
        # each rank on its own (instance) stream: ranks sharing a device in one process must not
        # meet on the legacy default stream, where one rank's waiting exchange kernel would block
        # the other rank's work queued behind it
        with torch.cuda.stream(torch.cuda.ExternalStream(di.inst.stream())):
            try:
                op = fg.krylov.DistOperator(di)
                b = 0.5 + 1e-3 * (plan.test_global % 89)
                b_loc = torch.from_numpy(b * plan.owned_mask).cuda()
                owned = torch.from_numpy(plan.owned_mask.astype(np.float64)).cuda()

                def dot(a, c):  # dist_cg's all-reduce, emulated with the thread gather
                    part = float(torch.dot(a * owned, c))
                    return torch.tensor(sum(gather(part)), dtype=torch.float64, device=a.device)

                def apply(v, out):
                    op.apply(v, out)
                    out.mul_(owned)  # ghost rows hold partial sums: only owned rows are the product
                x, it, _ = fg.krylov.cg(apply, b_loc, rtol=1e-10, maxiter=800, check_every=5, dot=dot)
                di.check()
                return plan.test_global[plan.owned_mask], x.cpu().numpy()[plan.owned_mask], it
            finally:
                di.close()

    res = run_ranks(world, rank)
    p = fg.symmetric_problem(*args)
    x = np.full(p.output_size, np.nan)
    for g, v, _ in res:
        x[g] = v
    assert not np.isnan(x).any()
    b = 0.5 + 1e-3 * (np.arange(p.output_size) % 89)
    p.scalar_inputs[0] = x
    assert np.linalg.norm(oracle.reference_action(p) - b) <= 1e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("world", [2, 3])
def test_native_distributed_cg_with_device_allreduce(oracle, world):
    """femgpu_halo_cg: the whole distributed CG on the devices, dots all-reduced GPU to GPU through the
    peers' flag words; the assembled solution satisfies the global A x = b."""
    import torch
    args = ("helmholtz", 3, 2, 14, 4)

    def rank(r, gather):
        slab = fdist.rank_slab(args, r, world)
        tab = slab.local.tabulations
        tab.psi = np.ascontiguousarray(np.transpose(tab.scalar_phi[0], (0, 2, 1)))
        plan = fdist.build_plan(slab, r, world, gather)
        di = fdist.DistInstance(plan, gather)
        try:
            b = 0.5 + 1e-3 * (plan.test_global % 89)
            b_loc = torch.from_numpy(b * plan.owned_mask).cuda()
            x, it, rel = di.cg(b_loc, rtol=1e-10, maxiter=800, check_every=5)
            di.check()
            return plan.test_global[plan.owned_mask], x.cpu().numpy()[plan.owned_mask], it, rel
        finally:
            di.close()

    res = run_ranks(world, rank)
    assert len({r[2] for r in res}) == 1  # every rank ran the same iterations (same all-reduced scalars)
    p = fg.symmetric_problem(*args)
    x = np.full(p.output_size, np.nan)
    for g, v, _, _ in res:
        x[g] = v
    assert not np.isnan(x).any()
    b = 0.5 + 1e-3 * (np.arange(p.output_size) % 89)
    p.scalar_inputs[0] = x
    assert np.linalg.norm(oracle.reference_action(p) - b) <= 1e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("config,n", [("C2", 12), ("C4", 8)])
def test_bench_launches_its_own_ranks_ipc_path(config, n):
    """bench.py --gpus 2 without torchrun launches its two ranks itself; they share cuda:0 through
    CUDA IPC (the cross-process path of csrc/halo.cu) and rank 0 checks the gathered owned rows
    against the reference CPU action."""
    env = dict(os.environ, FEMGPU_AUTOTUNE="0")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--config", config, "--mesh-n", str(n), "--steps", "5",
           "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-6000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["n_gpus"] == 2 and out["parity_complete"]
    assert out["parity_vs_reference"]["pass"], out["parity_vs_reference"]


@pytest.mark.parametrize("name,n", [("C2", 5), ("C4", 4)])
def test_halo_action_on_a_reordered_general_mesh(oracle, name, n):
    """A general mesh (cells shuffled, then femgpu_problem_reorder) split into contiguous Morton
    ranges (dist.problem_slab): the GPU-to-GPU exchange reproduces the reference action."""
    from tests.test_reorder import shuffled
    world = 2
    q, _ = fg.reorder_problem(shuffled(name, n))

    def rank(r, gather):
        plan = fdist.build_plan(fdist.problem_slab(q, r, world), r, world, gather)
        di = fdist.DistInstance(plan, gather)
        try:
            di.action()
            di.check()
            return di.owned_output()
        finally:
            di.close()

    res = run_ranks(world, rank)
    y = np.full(q.output_size, np.nan)
    for g, v in res:
        y[g] = v
    ref = oracle.reference_action(q)
    assert not np.isnan(y).any()
    assert rel_l2(y, ref) <= 1e-12 and max_rel(y, ref) <= 1e-10
