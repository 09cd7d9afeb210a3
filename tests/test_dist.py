"""Multi-process (gloo, world_size 2 and 3) tests of the cell-partitioned action: the partition
plan, DOF ownership and the forward/reverse halo exchanges of paper_2506_17471_b200/dist.py,
with the local compute done by the CPU oracle.  The GPU path uses the same plan and exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import dist as fdist
from tests.helpers import preset_problem, rel_l2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    kind, args = case
    p = fg.mesh_problem(*args) if kind == "mesh" else preset_problem(*args)
    gids, ys = fdist.cpu_action_with_halo(p, rank, world, oracle.reference_action)
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=gids, ys=ys)
    dist.barrier()
    dist.destroy_process_group()


CASES = [("mesh", ("laplace", 3, 2, 4, 4)), ("mesh", ("mass", 2, 1, 3, 12)), ("mesh", ("elasticity", 3, 2, 4, 3)),
         ("mesh", ("helmholtz_coef", 2, 3, 12, 6)), ("preset", ("laplace", 2, 2, 6, 48, 7))]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(str(a) for a in c[1]))
def test_partitioned_action_matches_oracle(tmp_path, case, world):
    from oracle import oracle
    port = _free_port()
    mp.spawn(_worker, args=(world, port, case, str(tmp_path)), nprocs=world, join=True)
    kind, args = case
    p = fg.mesh_problem(*args) if kind == "mesh" else preset_problem(*args)
    ref = oracle.reference_action(p)
    y = np.full(p.output_size, np.nan)
    for r in range(world):
        d = np.load(os.path.join(tmp_path, "r%d.npz" % r))
        assert np.all(np.isnan(y[d["gids"]])), "a DOF is owned by two ranks"
        y[d["gids"]] = d["ys"]
    assert not np.any(np.isnan(y)), "a DOF has no owner"
    assert rel_l2(y, ref) <= 1e-12


def test_split_cells_aligned_and_complete():
    for cells, world in [(6 * 1000, 8), (6 * 7, 3), (12, 5)]:
        r = fdist.split_cells(cells, world, 6)
        assert r[0][0] == 0 and r[-1][1] == cells
        for (b0, e0), (b1, e1) in zip(r, r[1:]):
            assert e0 == b1
        assert all(b % 6 == 0 for b, _ in r)


def test_ownership_is_lowest_rank():
    p = fg.mesh_problem("laplace", 3, 2, 4, 4)
    plans = fdist.plan(p, 3)
    owner = {}
    for pl in plans:
        for g in pl.test_global[pl.owned_mask]:
            assert g not in owner
            owner[g] = pl.rank
    for pl in plans:
        for g in pl.test_global:
            assert owner[g] <= pl.rank
