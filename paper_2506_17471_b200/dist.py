"""Cell-partitioned multi-GPU action: one process per GPU, torch.distributed
(NCCL on GPUs, gloo for CPU tests) for the plumbing.

Partition: rank r owns the contiguous cell range [c_r, c_{r+1}) of the brick-major cell order
(z-slabs of bricks on the structured meshes), aligned to the macro-element group size so every
rank keeps the compile-time connectivity pattern.  Each rank renumbers the DOFs/vertices its
cells touch (ascending global index) into a compact local instance.

Ownership: a DOF is owned by the lowest rank touching it.  Per action:
  1. forward halo: owners send x on shared DOFs to the ranks that also touch them;
  2. local action on the GPU (femgpu kernels) into the local y;
  3. reverse halo: non-owners send their partial y on shared DOFs to the owner, which adds
     them in ascending rank order (deterministic).
Only interface DOFs move (z-slab interfaces: ~(2N+1)^2 DOFs per neighbour for P2), so the
exchange is point-to-point send/recv, not an allreduce.
"""
from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

from .form import IndexMap, MeshConnectivity, ProblemInstance


@dataclass
class RankPlan:
    rank: int
    cell_range: tuple
    local: ProblemInstance                      # compact local instance
    test_global: np.ndarray                     # local test DOF -> global
    trial_global: List[np.ndarray]              # per trial space (scalar then vector): local node -> global
    owned_mask: np.ndarray                      # local test DOFs this rank owns
    # reverse halo (y): to owner q: local indices (sorted by global id); from rank q: local indices
    y_send: Dict[int, np.ndarray] = field(default_factory=dict)
    y_recv: Dict[int, np.ndarray] = field(default_factory=dict)
    # forward halo (x of trial space 0): owner -> ghosts
    x_send: Dict[int, np.ndarray] = field(default_factory=dict)
    x_recv: Dict[int, np.ndarray] = field(default_factory=dict)


def split_cells(cells: int, nranks: int, align: int = 6) -> List[tuple]:
    """Contiguous ranges, boundaries aligned to `align` cells (macro-element group size)."""
    units = (cells + align - 1) // align
    out = []
    for r in range(nranks):
        b = min(cells, (units * r // nranks) * align)
        e = min(cells, (units * (r + 1) // nranks) * align)
        out.append((b, e))
    return out


def _compact(m: np.ndarray):
    uniq, inv = np.unique(m, return_inverse=True)
    return uniq.astype(np.int64), inv.reshape(m.shape).astype(np.int32)


def local_instance(p: ProblemInstance, b: int, e: int):
    """Compact sub-instance of cells [b, e) (same restriction as the reference harness)."""
    sig, conn = p.signature, p.connectivity
    lc = MeshConnectivity(cell_count=e - b)
    trial_global, sx, vx = [], [], []
    cache = {}

    def comp(im: IndexMap):
        key = id(im.indices)
        if key not in cache:
            cache[key] = _compact(im.indices[b:e])
        return cache[key]

    for im, x in zip(conn.scalar_maps, p.scalar_inputs):
        u, loc = comp(im)
        lc.scalar_maps.append(IndexMap(loc, len(u)))
        sx.append(np.ascontiguousarray(x[u]))
        trial_global.append(u)
    for im, x in zip(conn.vector_maps, p.vector_inputs):
        u, loc = comp(im)
        lc.vector_maps.append(IndexMap(loc, len(u)))
        d = sig.dim
        vx.append(np.ascontiguousarray(x.reshape(-1, d)[u].reshape(-1)))
        trial_global.append(u)
    ut, loct = comp(conn.test_map)
    lc.test_map = IndexMap(loct, len(ut))
    if sig.affine_geometry:
        uc, locc = comp(conn.coord_map)
        lc.coord_map = IndexMap(locc, len(uc))
        lc.coords = np.ascontiguousarray(conn.coords[uc])
        lc.coord_global_count = len(uc)
    q = ProblemInstance(sig, p.map, p.tabulations, lc, sx, vx, len(ut))
    q.validate()
    return q, ut, trial_global


def plan(p: ProblemInstance, nranks: int, align: int = 6) -> List[RankPlan]:
    ranges = split_cells(p.connectivity.cell_count, nranks, align)
    plans = []
    for r, (b, e) in enumerate(ranges):
        loc, tg, trg = local_instance(p, b, e)
        plans.append(RankPlan(r, (b, e), loc, tg, trg, np.zeros(len(tg), dtype=bool)))
    # owner of each global test DOF = lowest rank touching it
    owner = np.full(p.output_size, nranks, dtype=np.int64)
    for pl in reversed(plans):
        owner[pl.test_global] = pl.rank
    for pl in plans:
        pl.owned_mask = owner[pl.test_global] == pl.rank
    for pl in plans:
        for q in plans:
            if q.rank == pl.rank:
                continue
            common, ia, ib = np.intersect1d(pl.test_global, q.test_global, assume_unique=True, return_indices=True)
            if common.size == 0:
                continue
            # reverse (y): pl -> owner q when q owns; forward (x): owner pl -> q
            mine_to_q = owner[common] == q.rank
            if mine_to_q.any():
                pl.y_send[q.rank] = ia[mine_to_q].astype(np.int64)
                q.y_recv[pl.rank] = ib[mine_to_q].astype(np.int64)
            if p.signature.scalar_spaces and np.array_equal(p.connectivity.scalar_maps[0].indices,
                                                            p.connectivity.test_map.indices):
                owned_by_pl = owner[common] == pl.rank
                if owned_by_pl.any():
                    pl.x_send[q.rank] = ia[owned_by_pl].astype(np.int64)
                    q.x_recv[pl.rank] = ib[owned_by_pl].astype(np.int64)
    return plans


def exchange(plan_: RankPlan, buf, send: Dict[int, np.ndarray], recv: Dict[int, np.ndarray], add: bool, xp):
    """Point-to-point halo exchange on torch tensors (NCCL or gloo): send buf[send[q]] to q,
    receive into buf[recv[q]] (added in ascending rank order when add=True)."""
    import torch.distributed as dist
    if buf.is_cuda and dist.get_backend() == "gloo":
        # gloo moves host tensors only: stage through the host (tests run several ranks on one GPU)
        host = buf.detach().cpu()
        cpu = lambda d: {q: (v.cpu() if hasattr(v, "cpu") else v) for q, v in d.items()}  # noqa: E731
        exchange(plan_, host, cpu(send), cpu(recv), add, xp)
        buf.copy_(host.to(buf.device))
        return buf
    ops, recvs = [], []
    for q in sorted(set(send) | set(recv)):
        if q in send:
            ops.append(dist.P2POp(dist.isend, buf[send[q]].contiguous(), q))
        if q in recv:
            t = xp.empty(len(recv[q]), dtype=buf.dtype, device=buf.device)
            recvs.append((q, t))
            ops.append(dist.P2POp(dist.irecv, t, q))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for q, t in sorted(recvs, key=lambda x: x[0]):
        if add:
            buf.index_add_(0, recv[q], t)
        else:
            buf[recv[q]] = t
    return buf


def _index_tensors(pl: RankPlan, device):
    import torch
    conv = lambda d: {q: torch.as_tensor(v, device=device) for q, v in d.items()}  # noqa: E731
    return conv(pl.y_send), conv(pl.y_recv), conv(pl.x_send), conv(pl.x_recv)


class _CudaArray:
    """Zero-copy torch view of a libfemgpu device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


def bench(args):
    """Multi-GPU bench leg (torchrun): strong scaling of the C2 action on the fixed mesh."""
    import torch
    import torch.distributed as dist

    import paper_2506_17471_b200 as fg
    from paper_2506_17471_b200._native import lib

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    device = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    backend = os.environ.get("FEMGPU_DIST_BACKEND", "nccl")  # gloo: functional tests with ranks sharing a GPU
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))
    else:
        dist.init_process_group(backend)
    lib().femgpu_set_device(device)
    p = fg.config_problem(args.config, n=args.n)
    plans = plan(p, world)
    pl = plans[rank]
    g = fg.GpuInstance(pl.local)
    dev = torch.device("cuda", device)
    ysend, yrecv, xsend, xrecv = _index_tensors(pl, dev)
    y = torch.zeros(pl.local.output_size, dtype=torch.float64, device=dev)
    import ctypes as C
    x = None
    if pl.x_send or pl.x_recv:
        # forward halo of trial space 0 (scalar, same numbering as the test space)
        xp = C.c_void_p()
        lib().femgpu_device_input(g.handle, 0, C.byref(xp))
        x = torch.as_tensor(_CudaArray(xp.value, pl.local.scalar_inputs[0].size), device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if x is not None:
            exchange(pl, x, xsend, xrecv, False, torch)
        g.action_device(y_dev=y.data_ptr(), stream=stream.cuda_stream or 1)
        exchange(pl, y, ysend, yrecv, True, torch)

    for _ in range(max(args.warmup, 3)):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / args.steps], dtype=torch.float64,
                     device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_step = float(t.item())
    # parity: gather owned y to rank 0 and compare with the single-instance GPU result
    gdev = dev if backend == "nccl" else torch.device("cpu")  # gloo collectives on host tensors
    owned = y[torch.as_tensor(np.nonzero(pl.owned_mask)[0], device=dev)].to(gdev)
    gids = torch.as_tensor(pl.test_global[pl.owned_mask], device=gdev)
    sizes = [None] * world
    dist.all_gather_object(sizes, int(owned.numel()))
    mx = max(sizes)
    pad = lambda t: torch.cat([t, t.new_zeros(mx - t.numel())])  # noqa: E731  (all_gather needs equal sizes)
    outs = [torch.empty(mx, dtype=torch.float64, device=gdev) for _ in sizes]
    ids = [torch.empty(mx, dtype=torch.int64, device=gdev) for _ in sizes]
    dist.all_gather(outs, pad(owned))
    dist.all_gather(ids, pad(gids))
    outs = [o[:s] for o, s in zip(outs, sizes)]
    ids = [i[:s] for i, s in zip(ids, sizes)]
    if rank == 0:
        yfull = np.zeros(p.output_size)
        for o, i in zip(outs, ids):
            yfull[i.cpu().numpy()] = o.cpu().numpy()
        halo = sum(len(v) for v in pl.y_send.values()) + sum(len(v) for v in pl.y_recv.values())
        out = {
            "metric": "FP64 operator-action GDOF/s", "value": p.output_size / t_step / 1e9, "unit": "GDOF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s cell-partitioned over %d GPUs (contiguous brick-major ranges), %s"
                                   "action + reverse y halo over %s per step"
                                   % (args.config, world, "forward x halo + " if x is not None else
                                      "(x static: no forward halo planned for this trial space) + ", backend.upper()),
                       "cells": int(p.connectivity.cell_count), "dofs": int(p.output_size),
                       "rank0_halo_dofs": int(halo), "parallelism": "cells%d" % world},
            "gpu_launches": args.steps,
        }
        with fg.GpuInstance(p) as gi:
            ref = gi.action()
        out["parity_vs_1gpu_rel_l2"] = float(np.linalg.norm(yfull - ref) / np.linalg.norm(ref))
        out["backend"] = backend
        print(json.dumps(out))
    dist.destroy_process_group()
    g.close()


def cpu_action_with_halo(p: ProblemInstance, rank: int, world: int, action):
    """CPU leg for the gloo tests: the same plan and exchange, local compute by `action`
    (the oracle), returning (owned global ids, owned y)."""
    import torch
    plans = plan(p, world)
    pl = plans[rank]
    ys, yr, xs, xr = (
        {q: torch.as_tensor(v) for q, v in d.items()} for d in (pl.y_send, pl.y_recv, pl.x_send, pl.x_recv))
    x = torch.as_tensor(pl.local.scalar_inputs[0].copy()) if pl.local.scalar_inputs else None
    if x is not None:
        # ghosts start stale (zero) and must be filled by the forward halo from the owners
        ghost = np.concatenate([v for v in pl.x_recv.values()]) if pl.x_recv else np.zeros(0, dtype=np.int64)
        x[torch.as_tensor(ghost)] = 0.0
        exchange(pl, x, xs, xr, False, torch)
        pl.local.scalar_inputs[0] = x.numpy().copy()
    y = torch.as_tensor(action(pl.local))
    exchange(pl, y, ys, yr, True, torch)
    m = pl.owned_mask
    return pl.test_global[m], y.numpy()[m]
