"""The CG caller (paper_2506_17471_b200/krylov.py).

CPU: the CG algorithm on torch CPU tensors with the CPU oracle as the operator (symmetric Helmholtz
instance, Psi = Phi^T) converges and its solution satisfies the oracle's A x = b.
GPU: the device-resident loop (femgpu_action_device into torch tensors, no host copies per action)
converges to the same tolerance, checked against the oracle's action."""
import numpy as np
import pytest
import torch

import paper_2506_17471_b200 as fg


def oracle_apply(oracle, p):
    def apply(v, out):
        p.scalar_inputs[0] = v.numpy().copy()
        out.copy_(torch.from_numpy(oracle.reference_action(p)))
    return apply


def test_symmetric_problem_is_symmetric(oracle):
    p = fg.symmetric_problem("helmholtz", 2, 2, 6, 3)
    n = p.output_size
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    p.scalar_inputs[0] = u
    au = oracle.reference_action(p)
    p.scalar_inputs[0] = v
    av = oracle.reference_action(p)
    assert abs(np.dot(v, au) - np.dot(u, av)) <= 1e-12 * np.linalg.norm(au) * np.linalg.norm(v)


def test_cg_converges_with_oracle_operator(oracle):
    p = fg.symmetric_problem("helmholtz", 2, 2, 6, 4)
    b = torch.from_numpy(np.random.default_rng(3).uniform(0.5, 1.5, p.output_size))
    x, it, hist = fg.cg(oracle_apply(oracle, p), b, rtol=1e-10, maxiter=500)
    assert hist[-1] <= 1e-10 * float(torch.linalg.norm(b)) and it < 500
    p.scalar_inputs[0] = x.numpy().copy()
    r = oracle.reference_action(p) - b.numpy()
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(b.numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("form,dim,deg,Q,n", [("helmholtz", 3, 2, 14, 4), ("mass", 3, 2, 14, 4)])
def test_device_cg_converges(oracle, form, dim, deg, Q, n):
    p = fg.symmetric_problem(form, dim, deg, Q, n)
    dev = torch.device("cuda", 0)
    b = torch.from_numpy(np.random.default_rng(5).uniform(0.5, 1.5, p.output_size)).to(dev)
    with fg.GpuInstance(p) as g:
        op = fg.DeviceOperator(g)
        x, it, hist = fg.cg(op.apply, b, rtol=1e-10, maxiter=2000, check_every=5)
        assert op.launches == it  # one device action per iteration, no extra launches
    assert hist[-1] <= 1e-10 * float(torch.linalg.norm(b))
    p.scalar_inputs[0] = x.cpu().numpy().copy()
    r = oracle.reference_action(p) - b.cpu().numpy()
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("form,dim,deg,Q,n", [("helmholtz", 3, 2, 14, 4), ("laplace", 3, 2, 4, 5), ("mass", 2, 3, 12, 8)])
def test_native_cg_converges_and_is_reproducible(oracle, form, dim, deg, Q, n):
    """femgpu_cg (csrc/cg.cu): the loop inside libfemgpu converges to the oracle's solution and needs
    about the iterations of the torch loop; a second solve agrees to rounding (the reductions are
    fixed-order, the action's red.add scatter is not)."""
    p = fg.symmetric_problem(form, dim, deg, Q, n)
    if form == "laplace":  # Laplace is only semi-definite: shift by the mass-like Helmholtz term instead
        p = fg.symmetric_problem("helmholtz", dim, deg, Q, n)
    dev = torch.device("cuda", 0)
    b = torch.from_numpy(np.random.default_rng(5).uniform(0.5, 1.5, p.output_size)).to(dev)
    with fg.GpuInstance(p) as g:
        x, it, rel = fg.krylov.native_cg(g, b, rtol=1e-10, maxiter=3000, check_every=1)
        x2, it2, rel2 = fg.krylov.native_cg(g, b, rtol=1e-10, maxiter=3000, check_every=1)
        # residual checks every 10 iterations: the iterations between checks replay as a CUDA graph
        x3, it3, rel3 = fg.krylov.native_cg(g, b, rtol=1e-10, maxiter=3000, check_every=10)
        op = fg.DeviceOperator(g)
        _, it_t, _ = fg.cg(op.apply, b, rtol=1e-10, maxiter=3000, check_every=1)
    assert rel <= 1e-10 and it < 3000
    assert abs(it - it2) <= 2 and float(torch.linalg.norm(x - x2) / torch.linalg.norm(x)) <= 1e-9
    assert rel3 <= 1e-10 and it - 2 <= it3 <= it + 12 and float(torch.linalg.norm(x - x3) / torch.linalg.norm(x)) <= 1e-8
    assert abs(it - it_t) <= max(2, it_t // 20)
    p.scalar_inputs[0] = x.cpu().numpy().copy()
    r = oracle.reference_action(p) - b.cpu().numpy()
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b.cpu().numpy())


def _dist_worker(rank, world, port, out_dir):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2506_17471_b200 import dist as fdist
    slab = fdist.rank_slab(("helmholtz", 2, 2, 6, 6), rank, world)
    tab = slab.local.tabulations
    tab.psi = np.ascontiguousarray(np.transpose(tab.scalar_phi[0], (0, 2, 1)))  # as symmetric_problem
    pl = fdist.build_plan(slab, rank, world, fdist.torch_gather())
    b = np.random.default_rng(3).uniform(0.5, 1.5, (2 * 6 + 1) ** 2)

    def dist_apply(v, out):  # pull ghosts, local oracle action, push partial rows (host emulation)
        out.copy_(torch.from_numpy(fdist.host_halo_action(pl, oracle.reference_action, [v.numpy().copy()])))

    b_loc = torch.from_numpy(b[pl.test_global] * pl.owned_mask)
    x, it, hist = fg.krylov.dist_cg(pl, dist_apply, b_loc, rtol=1e-10, maxiter=500)
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=pl.test_global[pl.owned_mask],
             xs=x.numpy()[pl.owned_mask], it=it)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_cg_matches_single_process(tmp_path, oracle, world):
    import os
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_dist_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    p = fg.symmetric_problem("helmholtz", 2, 2, 6, 6)
    b = np.random.default_rng(3).uniform(0.5, 1.5, p.output_size)
    x = np.full(p.output_size, np.nan)
    for r in range(world):
        d = np.load(os.path.join(tmp_path, "r%d.npz" % r))
        x[d["gids"]] = d["xs"]
    assert not np.any(np.isnan(x))
    p.scalar_inputs[0] = x
    res = oracle.reference_action(p) - b
    assert np.linalg.norm(res) <= 1e-9 * np.linalg.norm(b)


@pytest.mark.gpu
def test_native_cg_rejects_non_square_operators():
    p = fg.mesh_problem("helmholtz_coef", 2, 3, 12, 4)  # two scalar spaces: not a square scalar operator
    b = torch.ones(p.output_size, dtype=torch.float64, device="cuda")
    with fg.GpuInstance(p) as g:
        with pytest.raises(ValueError, match="cg:"):
            fg.krylov.native_cg(g, b)
