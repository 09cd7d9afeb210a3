"""CPU tests of the cell-partitioned action (paper_2506_17471_b200/dist.py): per-rank slabs built
without the global mesh, the collective discovery/ownership plan, and the exchange it prescribes,
emulated on the host over gloo (world size 2 and 3) with the CPU oracle as local compute.  The GPU
path (csrc/halo.cu) executes the same plan GPU to GPU (tests/test_gpu_dist.py)."""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import dist as fdist
from tests.helpers import rel_l2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class ThreadGather:
    """all-gather among `world` threads of one process (the collective plan without processes)."""

    def __init__(self, world):
        self.world, self.slots, self.bar = world, [None] * world, threading.Barrier(world)

    def for_rank(self, r):
        def gather(obj):
            self.slots[r] = obj
            self.bar.wait()
            out = list(self.slots)
            self.bar.wait()
            return out
        return gather


def plans_in_threads(args, world):
    tg = ThreadGather(world)
    plans = [None] * world

    def run(r):
        plans[r] = fdist.build_plan(fdist.rank_slab(args, r, world), r, world, tg.for_rank(r))
    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return plans


FORMS = [("laplace", 3, 2, 4, 4), ("mass", 2, 1, 3, 12), ("elasticity", 3, 2, 4, 3),
         ("helmholtz_coef", 2, 3, 12, 6), ("hyperelastic", 3, 1, 4, 3), ("advection", 3, 2, 14, 2)]


@pytest.mark.parametrize("args", FORMS, ids=lambda a: "-".join(map(str, a)))
def test_slab_equals_restriction_of_the_global_instance(args):
    """A rank's slab (femgpu_mesh_build_range + counter-based draws) is the compact restriction of
    the global instance to its cells: same maps, inputs, coordinates, tabulations."""
    p = fg.mesh_problem(*args)
    for world in (2, 3):
        for r, (b, e) in enumerate(fdist.split_cells(p.connectivity.cell_count, world, fdist.group_align(args[1]))):
            s = fdist.rank_slab(args, r, world)
            q, _, _ = fdist.local_instance(p, b, e)
            a, c = s.local, q
            assert a.output_size == c.output_size
            assert np.array_equal(a.connectivity.test_map.indices, c.connectivity.test_map.indices)
            for m1, m2 in zip(a.connectivity.scalar_maps + a.connectivity.vector_maps,
                              c.connectivity.scalar_maps + c.connectivity.vector_maps):
                assert np.array_equal(m1.indices, m2.indices) and m1.global_count == m2.global_count
            for x1, x2 in zip(a.scalar_inputs + a.vector_inputs, c.scalar_inputs + c.vector_inputs):
                assert np.array_equal(x1, x2)
            assert np.array_equal(a.connectivity.coords, c.connectivity.coords)
            assert np.array_equal(a.tabulations.psi, c.tabulations.psi)


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("args", FORMS[:4], ids=lambda a: "-".join(map(str, a)))
def test_plan_is_consistent_across_ranks(args, world):
    """Every row has exactly one owner (the lowest rank touching it); r's push list to q and q's
    receive list from r name the same global rows in the same order; every pulled node maps to the
    same global node at its owner; boundary-first cell order with all shared rows in the boundary."""
    plans = plans_in_threads(args, world)
    owner = {}
    for pl in plans:
        for g in pl.test_global[pl.owned_mask]:
            assert g not in owner
            owner[int(g)] = pl.rank
    for pl in plans:
        for g in pl.test_global:
            assert owner[int(g)] <= pl.rank
        for q, rows in pl.push.items():
            theirs = plans[q].recv[pl.rank]
            assert np.array_equal(pl.test_global[rows], plans[q].test_global[theirs])
            assert all(owner[int(g)] == q for g in pl.test_global[rows])
        for s, d in enumerate(pl.pull):
            for q, (mine, remote) in d.items():
                assert np.array_equal(pl.trial_global[s][mine], plans[q].trial_global[s][remote])
                assert np.array_equal(np.sort(plans[q].serve[s][pl.rank]), np.sort(remote))
        shared = np.zeros(pl.local.output_size, dtype=bool)
        for v in list(pl.push.values()) + list(pl.recv.values()):
            shared[v] = True
        tm = pl.local.connectivity.test_map.indices
        touching = np.nonzero(shared[tm].any(axis=1))[0]
        assert touching.size == 0 or touching.max() < pl.boundary_cells


def _worker(rank, world, port, args, out_dir, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    if mode == "action":
        gids, ys = fdist.cpu_action_with_halo(args, rank, world, oracle.reference_action)
        np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=gids, ys=ys)
    else:  # changing inputs: owned values set from the new global x, ghosts poisoned (NaN)
        plan = fdist.build_plan(fdist.rank_slab(args, rank, world), rank, world, fdist.torch_gather())
        p = plan.local
        ns = len(p.scalar_inputs)
        d = p.signature.dim
        for step in range(2):
            xs = []
            for s, gl in enumerate(plan.trial_global):
                comps = 1 if s < ns else d
                own = np.full(len(gl), True)
                for q, (mine, _) in plan.pull[s].items():
                    own[mine] = False
                val = (0.5 + 0.25 * step + 1e-3 * ((gl[:, None] * comps + np.arange(comps)) % 97)).reshape(-1)
                val = val.reshape(len(gl), comps)
                val[~own] = np.nan
                xs.append(val.reshape(-1))
            y = fdist.host_halo_action(plan, oracle.reference_action, xs)
            m = plan.owned_mask
            np.savez(os.path.join(out_dir, "r%d_s%d.npz" % (rank, step)), gids=plan.test_global[m], ys=y[m])
    dist.barrier()
    dist.destroy_process_group()


def _general_worker(rank, world, port, name, n, out_dir):
    """A general mesh (cells shuffled, then femgpu_problem_reorder): contiguous Morton ranges per rank
    (dist.problem_slab), the collective plan and the host exchange with the oracle as local compute."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from tests.test_reorder import shuffled
    q, _ = fg.reorder_problem(shuffled(name, n))
    plan = fdist.build_plan(fdist.problem_slab(q, rank, world), rank, world, fdist.torch_gather())
    y = fdist.host_halo_action(plan, oracle.reference_action)
    m = plan.owned_mask
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=plan.test_global[m], ys=y[m])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C2", 4), ("C4", 3)])
def test_general_mesh_partition_after_reorder(tmp_path, name, n):
    from oracle import oracle
    from tests.test_reorder import shuffled
    world = 3
    mp.spawn(_general_worker, args=(world, _free_port(), name, n, str(tmp_path)), nprocs=world, join=True)
    q, _ = fg.reorder_problem(shuffled(name, n))
    assert rel_l2(_assemble(str(tmp_path), world, q.output_size), oracle.reference_action(q)) <= 1e-12


def _assemble(out_dir, world, n, suffix=""):
    y = np.full(n, np.nan)
    for r in range(world):
        dd = np.load(os.path.join(out_dir, "r%d%s.npz" % (r, suffix)))
        assert np.all(np.isnan(y[dd["gids"]])), "a DOF is owned by two ranks"
        y[dd["gids"]] = dd["ys"]
    assert not np.any(np.isnan(y)), "a DOF has no owner (or a ghost input was never pulled)"
    return y


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("args", FORMS[:4], ids=lambda a: "-".join(map(str, a)))
def test_partitioned_action_matches_oracle(tmp_path, args, world):
    from oracle import oracle
    mp.spawn(_worker, args=(world, _free_port(), args, str(tmp_path), "action"), nprocs=world, join=True)
    p = fg.mesh_problem(*args)
    assert rel_l2(_assemble(str(tmp_path), world, p.output_size), oracle.reference_action(p)) <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("args", [("elasticity", 3, 2, 4, 3), ("hyperelastic", 3, 1, 4, 3),
                                  ("helmholtz_coef", 2, 3, 12, 6)], ids=lambda a: "-".join(map(str, a)))
def test_forward_halo_refreshes_changed_inputs(tmp_path, args, world):
    """Inputs change between actions (every trial space, vector spaces included): each rank holds
    current values only on the nodes it owns and NaN on its ghosts; the forward halo must fill them."""
    from oracle import oracle
    mp.spawn(_worker, args=(world, _free_port(), args, str(tmp_path), "changing"), nprocs=world, join=True)
    p = fg.mesh_problem(*args)
    d = p.signature.dim
    for step in range(2):
        for i, x in enumerate(p.scalar_inputs):
            g = np.arange(len(x))
            p.scalar_inputs[i] = 0.5 + 0.25 * step + 1e-3 * (g % 97)
        for i, x in enumerate(p.vector_inputs):
            g = np.arange(len(x) // d)
            p.vector_inputs[i] = (0.5 + 0.25 * step + 1e-3 * ((g[:, None] * d + np.arange(d)) % 97)).reshape(-1)
        y = _assemble(str(tmp_path), world, p.output_size, "_s%d" % step)
        assert rel_l2(y, oracle.reference_action(p)) <= 1e-12, step


def _cg_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    slab = fdist.rank_slab(("helmholtz", 3, 2, 14, 3), rank, world)
    tab = slab.local.tabulations
    tab.psi = np.ascontiguousarray(np.transpose(tab.scalar_phi[0], (0, 2, 1)))  # symmetric (krylov.symmetric_problem)
    plan = fdist.build_plan(slab, rank, world, fdist.torch_gather())
    b = 0.5 + 1e-3 * (plan.test_global % 89)
    b_loc = torch.from_numpy(b * plan.owned_mask)

    def dist_apply(v, out):
        out[:] = torch.from_numpy(fdist.host_halo_action(plan, oracle.reference_action, [v.numpy().copy()]))
    x, it, hist = fg.krylov.dist_cg(plan, dist_apply, b_loc, rtol=1e-10, maxiter=500, check_every=5)
    m = plan.owned_mask
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=plan.test_global[m], ys=x.numpy()[m])
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_cg_solves_the_global_system(tmp_path):
    from oracle import oracle
    mp.spawn(_cg_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    p = fg.symmetric_problem("helmholtz", 3, 2, 14, 3)
    x = _assemble(str(tmp_path), 2, p.output_size)
    b = 0.5 + 1e-3 * (np.arange(p.output_size) % 89)
    p.scalar_inputs[0] = x
    assert np.linalg.norm(oracle.reference_action(p) - b) <= 1e-8 * np.linalg.norm(b)


def test_split_cells_aligned_and_complete():
    for cells, world in [(6 * 1000, 8), (6 * 7, 3), (12, 5)]:
        r = fdist.split_cells(cells, world, 6)
        assert r[0][0] == 0 and r[-1][1] == cells
        for (b0, e0), (b1, e1) in zip(r, r[1:]):
            assert e0 == b1
        assert all(b % 6 == 0 for b, _ in r)
