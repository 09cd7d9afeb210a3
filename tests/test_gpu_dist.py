"""End-to-end multi-process run of the multi-GPU bench path (bench.py under torch.distributed.run,
paper_2506_17471_b200/dist.py) on the one GPU this environment provides: two ranks share cuda:0 and
exchange halos over gloo (FEMGPU_DIST_BACKEND=gloo; NCCL refuses two ranks on one device).  Checks the
partitioned action (local GPU kernels + reverse y halo, forward x halo where planned) against the
single-instance GPU result: rel L2 <= 1e-12.  The NCCL transport itself needs >= 2 GPUs."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("config,n", [("C2", 10), ("C4", 8), ("C3a", 40)])
def test_two_ranks_on_one_gpu_match_single_instance(config, n):
    env = dict(os.environ, FEMGPU_DIST_BACKEND="gloo", FEMGPU_AUTOTUNE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--config", config, "--mesh-n", str(n), "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[:6000]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 2 and out["backend"] == "gloo"
    assert out["parity_vs_1gpu_rel_l2"] <= 1e-12, out


def _cg_worker(rank, world, port, out_dir):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2506_17471_b200 as fg
    from paper_2506_17471_b200 import dist as fdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p = fg.symmetric_problem("helmholtz", 3, 2, 14, 4)
    b = np.random.default_rng(3).uniform(0.5, 1.5, p.output_size)
    pl = fdist.plan(p, world)[rank]
    dev = torch.device("cuda", 0)
    with fg.GpuInstance(pl.local) as g:
        op = fg.DeviceOperator(g)
        b_loc = torch.from_numpy(b[pl.test_global] * pl.owned_mask).to(dev)
        x, it, hist = fg.krylov.dist_cg(pl, op.apply, b_loc, rtol=1e-10, maxiter=2000, check_every=5)
        np.savez(os.path.join(out_dir, "r%d.npz" % rank), gids=pl.test_global[pl.owned_mask],
                 xs=x.cpu().numpy()[pl.owned_mask], it=it, launches=op.launches)
    dist.barrier()
    dist.destroy_process_group()


def test_distributed_device_cg_two_ranks_one_gpu(tmp_path, oracle):
    """dist_cg with the local action on the GPU (DeviceOperator) and halos over gloo, two ranks on
    cuda:0: the assembled solution satisfies the oracle's A x = b."""
    import numpy as np
    import torch.multiprocessing as mp

    import paper_2506_17471_b200 as fg
    mp.spawn(_cg_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    p = fg.symmetric_problem("helmholtz", 3, 2, 14, 4)
    b = np.random.default_rng(3).uniform(0.5, 1.5, p.output_size)
    x = np.full(p.output_size, np.nan)
    for r in range(2):
        d = np.load(os.path.join(tmp_path, "r%d.npz" % r))
        x[d["gids"]] = d["xs"]
    assert not np.any(np.isnan(x))
    p.scalar_inputs[0] = x
    assert np.linalg.norm(oracle.reference_action(p) - b) <= 1e-8 * np.linalg.norm(b)
