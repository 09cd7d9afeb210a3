"""Cell-partitioned multi-GPU action: one process per GPU; torch.distributed (gloo) only
for the control plane (plan discovery, handle exchange, timing reduction); the data path is
GPU to GPU inside libfemgpu (csrc/halo.cu: NVLink loads/stores between ranks, device-side flags).

Partition: rank r owns the contiguous cell range [c_r, c_{r+1}) of the brick-major cell order
(z-slabs of bricks on the structured meshes), aligned to the macro-element group, and builds only
that slab (femgpu_mesh_build_range; inputs drawn at their global positions of the counter-based
SynthRng), renumbered compactly (ascending global index) into its own instance.

Discovery (collective, once): every rank publishes the global-index range of each of its maps;
ranks whose ranges overlap exchange the ids inside the overlap; a DOF/node is owned by the lowest
rank touching it.  From that each rank derives, in its local numbering:
  push   rows it computes partial sums for but does not own (per owner, ascending global id)
  recv   owned rows other ranks contribute to (per source, ascending global id: the same order)
  pull   ghost trial nodes and their index in the owner's instance (forward halo; every trial
         space, scalar or vector)
  serve  owned trial nodes other ranks pull (the owner's side of pull; host emulation only)
Cells touching a shared row are moved to the front of the local order (whole macro groups), so the
push overlaps the interior cells on the GPU.  The exchange volume is the slab interfaces only:
(2N+1)^2 P2 nodes per neighbour for C2 z-slabs.

The same plan drives a host emulation of the exchange (torch.distributed point-to-point, gloo) with
the local action done by any callable (the CPU oracle in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import abi
from .form import IndexMap, MeshConnectivity, ProblemInstance, SynthRng, _draw_tabulations, _seed0

# ------------------------------------------------------------------------------- partition


def split_cells(cells: int, nranks: int, align: int = 6) -> List[tuple]:
    """Contiguous ranges, boundaries aligned to `align` cells (macro-element group size)."""
    units = (cells + align - 1) // align
    out = []
    for r in range(nranks):
        b = min(cells, (units * r // nranks) * align)
        e = min(cells, (units * (r + 1) // nranks) * align)
        out.append((b, e))
    return out


def group_align(dim: int) -> int:
    return 6 if dim == 3 else 4  # one cube (6 Kuhn tets) / two squares: the macro groups


def _compact(m: np.ndarray):
    uniq, inv = np.unique(m, return_inverse=True)
    return uniq.astype(np.int64), inv.reshape(m.shape).astype(np.int32)


@dataclass
class Slab:
    """One rank's compact instance plus the global ids of its local numbering, per map kind."""
    local: ProblemInstance
    cell_range: tuple
    kinds: Dict[str, np.ndarray]          # map kind -> sorted global ids (local index = position)
    space_kind: List[str]                 # per trial space (scalar then vector): its map kind
    test_kind: str                        # "node", "vertex" or "node*d" (vector test space)
    dim: int


def slab_instance(form: str, dim: int, degree: int, Q: int, n: int, b: int, e: int, seed: int = 7,
                  brick: Optional[int] = None, scale_u0: float = 0.05) -> Slab:
    """Cells [b, e) of mesh_problem(form, dim, degree, Q, n, seed) built without the global mesh:
    the same maps (rows of femgpu_mesh_build), tabulations and input values (SynthRng draws at the
    global positions), compactly renumbered.  Equals local_instance(mesh_problem(...), b, e)."""
    from ._native import check, lib
    from .mesh import default_brick, form_map, form_signature, mesh_counts
    brick = default_brick(dim) if brick is None else brick
    sig = form_signature(form, dim, degree, Q)
    pmap = form_map(form, sig)
    _, n_nodes, n_verts, npc = mesh_counts(dim, n, degree)
    node_map = np.empty((e - b, npc), dtype=np.int32)
    vertex_map = np.empty((e - b, dim + 1), dtype=np.int32)
    check(lib().femgpu_mesh_build_range(dim, n, degree, brick, b, e, abi.iptr(node_map), abi.iptr(vertex_map), None))
    rng = SynthRng(_seed0(seed))
    tab = _draw_tabulations(sig, rng)
    nodes_u, nodes_loc = _compact(node_map)
    verts_u, verts_loc = _compact(vertex_map)
    kind_of = lambda dofs: "node" if dofs == npc else "vertex"  # noqa: E731  (as mesh_problem)
    glob = {"node": n_nodes, "vertex": n_verts}
    ids = {"node": nodes_u, "vertex": verts_u}
    loc = {"node": nodes_loc, "vertex": verts_loc}
    conn = MeshConnectivity(cell_count=e - b)
    sx, vx, space_kind = [], [], []
    off = 0
    for s in sig.scalar_spaces:
        k = kind_of(s.dofs)
        conn.scalar_maps.append(IndexMap(loc[k], len(ids[k])))
        sx.append(rng.uniform_at(0.25, 1.0, off + ids[k]))
        off += glob[k]
        space_kind.append(k)
    for i, v in enumerate(sig.vector_spaces):
        k = kind_of(v.dofs)
        conn.vector_maps.append(IndexMap(loc[k], len(ids[k])))
        pos = off + (ids[k][:, None] * dim + np.arange(dim)[None, :]).reshape(-1)
        x = rng.uniform_at(0.25, 1.0, pos)
        if form == "hyperelastic" and i == 1:
            x = x * scale_u0
        vx.append(x)
        off += glob[k] * dim
        space_kind.append(k)
    if sig.test_dofs == npc:
        conn.test_map, test_kind = IndexMap(nodes_loc, len(nodes_u)), "node"
    else:  # vector test space, node-major local order j = a*d + c (as mesh_problem)
        tm = (nodes_loc[:, :, None].astype(np.int64) * dim + np.arange(dim)[None, None, :]).reshape(e - b, npc * dim)
        conn.test_map, test_kind = IndexMap(tm.astype(np.int32), len(nodes_u) * dim), "node*d"
    conn.coord_map = IndexMap(verts_loc, len(verts_u))
    n1 = n + 1
    conn.coords = np.stack([((verts_u // n1 ** c) % n1) / n for c in range(dim)], axis=1).astype(np.float64)
    conn.coord_global_count = len(verts_u)
    p = ProblemInstance(sig, pmap, tab, conn, sx, vx, conn.test_map.global_count)
    p.validate()
    return Slab(p, (b, e), ids, space_kind, test_kind, dim)


def local_instance(p: ProblemInstance, b: int, e: int):
    """Compact sub-instance of cells [b, e) of a global instance (test reference for slab_instance,
    and the reference harness's per-thread restriction)."""
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


# ------------------------------------------------------------------------------- exchange plan


@dataclass
class RankPlan:
    rank: int
    world: int
    cell_range: tuple
    local: ProblemInstance            # cells ordered boundary-first
    boundary_cells: int
    test_global: np.ndarray           # local test row -> global row
    trial_global: List[np.ndarray]    # per trial space: local node -> global node
    owned_mask: np.ndarray            # local test rows this rank owns
    push: Dict[int, np.ndarray] = field(default_factory=dict)   # owner -> local rows (ascending global)
    recv: Dict[int, np.ndarray] = field(default_factory=dict)   # source -> owned local rows (same order)
    pull: List[Dict[int, Tuple[np.ndarray, np.ndarray]]] = field(default_factory=list)  # per space: owner -> (local, owner-local)
    serve: List[Dict[int, np.ndarray]] = field(default_factory=list)  # per space: puller -> owned local nodes

    def halo_rows(self) -> int:
        return int(sum(len(v) for v in self.push.values()) + sum(len(v) for v in self.recv.values()))


def _shared(my_ids: np.ndarray, their_ids: np.ndarray, their_pos: np.ndarray):
    """(global ids, my local positions, their local positions) of the common ids."""
    common, ia, ib = np.intersect1d(my_ids, their_ids, assume_unique=True, return_indices=True)
    return common, ia.astype(np.int64), their_pos[ib].astype(np.int64)


def discover(kinds: Dict[str, np.ndarray], rank: int, world: int, gather) -> Dict[str, Dict[int, tuple]]:
    """Per map kind: {q: (shared global ids, my positions, q's positions)} for every rank q sharing
    ids with this one.  `gather(obj)` all-gathers a picklable object over the ranks.  Only the ids
    inside overlapping global ranges travel (the slab interfaces on partitions with locality)."""
    rng = {k: (int(v[0]), int(v[-1])) if len(v) else (1, 0) for k, v in kinds.items()}
    ranges = gather(rng)
    offer = {}
    for k, ids in kinds.items():
        offer[k] = {}
        for q in range(world):
            if q == rank:
                continue
            lo, hi = ranges[q][k]
            if hi < lo or not len(ids):
                continue
            a, z = np.searchsorted(ids, lo), np.searchsorted(ids, hi, side="right")
            if z > a:
                offer[k][q] = (ids[a:z], np.arange(a, z, dtype=np.int64))
    offers = gather(offer)
    out = {}
    for k, ids in kinds.items():
        out[k] = {}
        for q in range(world):
            if q == rank or rank not in offers[q][k]:
                continue
            their_ids, their_pos = offers[q][k][rank]
            common, mine, theirs = _shared(ids, their_ids, their_pos)
            if common.size:
                out[k][q] = (common, mine, theirs)
    return out


def _owner_of(n_local: int, shared: Dict[int, tuple], rank: int) -> np.ndarray:
    owner = np.full(n_local, rank, dtype=np.int64)
    for q, (_, mine, _) in shared.items():
        owner[mine] = np.minimum(owner[mine], q)
    return owner


def _expand_rows(shared_nodes: Dict[int, tuple], dim: int) -> Dict[int, tuple]:
    """Node sharing -> row sharing of an interleaved vector test space (row = node*dim + c)."""
    out = {}
    for q, (g, mine, theirs) in shared_nodes.items():
        c = np.arange(dim)[None, :]
        out[q] = ((g[:, None] * dim + c).reshape(-1), (mine[:, None] * dim + c).reshape(-1),
                  (theirs[:, None] * dim + c).reshape(-1))
    return out


def build_plan(slab: Slab, rank: int, world: int, gather) -> RankPlan:
    """Collective: the exchange plan of this rank's slab (see the module docstring)."""
    p = slab.local
    shared = discover(slab.kinds, rank, world, gather)
    test_shared = shared["node"] if slab.test_kind == "node" else (
        shared["vertex"] if slab.test_kind == "vertex" else _expand_rows(shared["node"], slab.dim))
    if slab.test_kind == "node*d":
        test_global = (slab.kinds["node"][:, None] * slab.dim + np.arange(slab.dim)[None, :]).reshape(-1)
    else:
        test_global = slab.kinds[slab.test_kind]
    n_rows = p.output_size
    owner = _owner_of(n_rows, test_shared, rank)
    push, recv = {}, {}
    shared_row = np.zeros(n_rows, dtype=bool)
    for q, (g, mine, _) in sorted(test_shared.items()):
        shared_row[mine] = True
        order = np.argsort(g, kind="stable")
        mine = mine[order]
        to_q = owner[mine] == q
        if to_q.any():
            push[q] = mine[to_q]
        mine_owned = owner[mine] == rank
        if mine_owned.any():
            recv[q] = mine[mine_owned]
    # boundary-first cell order (whole macro groups: the compile-time group pattern survives)
    G = group_align(slab.dim)
    tm = p.connectivity.test_map.indices
    cells = tm.shape[0]
    touch = shared_row[tm].any(axis=1)
    if cells % G == 0:
        grp = touch.reshape(-1, G).any(axis=1)
        perm = np.concatenate([np.nonzero(grp)[0], np.nonzero(~grp)[0]])
        perm = (perm[:, None] * G + np.arange(G)[None, :]).reshape(-1)
        nb = int(grp.sum()) * G
    else:
        perm = np.arange(cells)
        nb = cells
    local = _permute_cells(p, perm)
    pull, serve, trial_global = [], [], []
    for s, k in enumerate(slab.space_kind):
        ids = slab.kinds[k]
        trial_global.append(ids)
        own = _owner_of(len(ids), shared[k], rank)
        ps, sv = {}, {}
        for q, (g, mine, theirs) in sorted(shared[k].items()):
            order = np.argsort(g, kind="stable")
            mine, theirs = mine[order], theirs[order]
            from_q = own[mine] == q
            if from_q.any():
                ps[q] = (mine[from_q], theirs[from_q])
            # q pulls from me the shared nodes I own (q > me: the owner is the lowest rank)
            q_ghost = own[mine] == rank
            if q_ghost.any() and q > rank:
                sv[q] = mine[q_ghost]
        pull.append(ps)
        serve.append(sv)
    return RankPlan(rank, world, slab.cell_range, local, nb, test_global, trial_global, owner == rank,
                    push, recv, pull, serve)


def _permute_cells(p: ProblemInstance, perm: np.ndarray) -> ProblemInstance:
    if np.array_equal(perm, np.arange(len(perm))):
        return p
    conn = p.connectivity
    c = MeshConnectivity(cell_count=conn.cell_count)
    c.scalar_maps = [IndexMap(np.ascontiguousarray(m.indices[perm]), m.global_count) for m in conn.scalar_maps]
    c.vector_maps = [IndexMap(np.ascontiguousarray(m.indices[perm]), m.global_count) for m in conn.vector_maps]
    c.test_map = IndexMap(np.ascontiguousarray(conn.test_map.indices[perm]), conn.test_map.global_count)
    if p.signature.affine_geometry:
        c.coord_map = IndexMap(np.ascontiguousarray(conn.coord_map.indices[perm]), conn.coord_map.global_count)
        c.coords = conn.coords
        c.coord_global_count = conn.coord_global_count
    q = ProblemInstance(p.signature, p.map, p.tabulations, c, p.scalar_inputs, p.vector_inputs, p.output_size)
    q.validate()
    return q


def config_slab(name: str, rank: int, world: int, n: Optional[int] = None, seed: int = 7) -> Slab:
    from .mesh import CONFIGS, mesh_counts
    c = dict(CONFIGS[name])
    if n is not None:
        c["n"] = n
    cells = mesh_counts(c["dim"], c["n"], c["degree"])[0]
    b, e = split_cells(cells, world, group_align(c["dim"]))[rank]
    return slab_instance(c["form"], c["dim"], c["degree"], c["Q"], c["n"], b, e, seed=seed)


def problem_slab(p: ProblemInstance, rank: int, world: int) -> Slab:
    """This rank's contiguous cell range of a general (already built) problem, e.g. a mesh renumbered
    by reorder.reorder_problem: Morton-ordered cells make contiguous ranges spatially compact, the
    partition SURVEY 8e names for general meshes.  Trial spaces must live on the test space's nodes
    ("node") or on the coordinate map's vertices ("vertex"), as the benchmark forms do."""
    C, d = p.connectivity.cell_count, p.signature.dim
    b, e = split_cells(C, world, 1)[rank]
    local, ut, trial_global = local_instance(p, b, e)
    conn = p.connectivity
    tm = conn.test_map.indices
    vec_test = p.signature.test_dofs != tm.shape[1] or any(
        m.indices.shape[1] * d == tm.shape[1] and np.array_equal(tm[:1], (m.indices[:1, :, None] * d + np.arange(d)).reshape(1, -1))
        for m in conn.vector_maps)
    node_map = None
    if vec_test:
        for m in conn.vector_maps:
            if m.indices.shape[1] * d == tm.shape[1] and np.array_equal(tm, (m.indices[:, :, None].astype(np.int64) * d
                                                                              + np.arange(d)).reshape(C, -1)):
                node_map = m.indices
        if node_map is None:
            raise ValueError("problem_slab: vector test space is not node*dim+comp of a vector trial space")
    else:
        node_map = tm
    nodes_u = np.unique(node_map[b:e]).astype(np.int64)
    kinds = {"node": nodes_u}
    if conn.coord_map is not None:
        kinds["vertex"] = np.unique(conn.coord_map.indices[b:e]).astype(np.int64)
    space_kind = []
    for im in conn.scalar_maps + conn.vector_maps:
        if np.array_equal(im.indices, node_map):
            space_kind.append("node")
        elif conn.coord_map is not None and np.array_equal(im.indices, conn.coord_map.indices):
            space_kind.append("vertex")
        else:
            raise ValueError("problem_slab: a trial space is neither on the test nodes nor on the vertices")
    return Slab(local, (b, e), kinds, space_kind, "node*d" if vec_test else "node", d)


def torch_gather():
    import torch.distributed as tdist

    def gather(obj):
        out = [None] * tdist.get_world_size()
        tdist.all_gather_object(out, obj)
        return out
    return gather


# ------------------------------------------------------------------------------- device path


class DistInstance:
    """One rank's GPU instance + its halo (femgpu_halo_*): distributed actions with the exchange
    GPU to GPU (csrc/halo.cu).  Collective construction (handle exchange over `gather`)."""

    def __init__(self, plan: RankPlan, gather):
        from . import action as fa
        from ._native import lib
        self.plan = plan
        self.inst = fa.GpuInstance(plan.local)
        # one schedule for every rank: rank 0 runs the automatic schedule on its slab (alone on the
        # device), the others take its decision, so all slabs run the same kernel
        sched = self.inst.default_schedule() if plan.rank == 0 else None
        self.params = gather(sched)[0]
        # JIT and every allocation before the first exchange: a module load or cudaMalloc may wait
        # for the device, which must never happen while a peer spins on this rank
        self.inst.action(self.params)
        L = lib()

        def cat(parts):
            return np.concatenate(parts) if parts else np.zeros(0)

        push_peer = cat([np.full(len(v), q) for q, v in sorted(plan.push.items())])
        push_row = cat([v for _, v in sorted(plan.push.items())])
        recv_peer = cat([np.full(len(v), q) for q, v in sorted(plan.recv.items())])
        recv_row = cat([v for _, v in sorted(plan.recv.items())])
        ps, pp, pn, pr = [], [], [], []
        for s, d in enumerate(plan.pull):
            for q, (mine, theirs) in sorted(d.items()):
                ps.append(np.full(len(mine), s))
                pp.append(np.full(len(mine), q))
                pn.append(mine)
                pr.append(theirs)
        self._keep = [np.ascontiguousarray(np.asarray(x, dtype=np.int32))
                      for x in (push_peer, push_row, recv_peer, recv_row, cat(ps), cat(pp), cat(pn), cat(pr))]
        ptr = [a.ctypes.data_as(C.POINTER(C.c_int32)) for a in self._keep]
        h = C.c_void_p()
        fa._call(L.femgpu_halo_create(self.inst.handle, plan.rank, plan.world, plan.boundary_cells,
                                      len(self._keep[0]), ptr[0], ptr[1], len(self._keep[2]), ptr[2], ptr[3],
                                      len(self._keep[4]), ptr[4], ptr[5], ptr[6], ptr[7], C.byref(h)))
        self.halo = h
        n = C.c_size_t()
        fa._call(L.femgpu_halo_export(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        fa._call(L.femgpu_halo_export(h, buf, n.value, C.byref(n)))
        blob = b"".join(gather(bytes(buf.raw)))
        fa._call(L.femgpu_halo_import(h, blob, n.value))
        gather(None)  # every rank has mapped its peers before anyone starts exchanging

    def action(self, params=None, y_dev: int = 0, stream: int = 0):
        from . import action as fa
        from ._native import lib
        sp = fa._sched(params if params is not None else self.params)
        fa._call(lib().femgpu_halo_action(self.halo, sp[0] if sp else None, C.c_void_p(y_dev), C.c_void_p(stream)))

    def time_steps(self, steps: int, params=None) -> float:
        from . import action as fa
        from ._native import lib
        s = C.c_double()
        sp = fa._sched(params if params is not None else self.params)
        fa._call(lib().femgpu_halo_time_steps(self.halo, sp[0] if sp else None, steps, C.byref(s)))
        return s.value

    def check(self, stream: int = 0):
        from . import action as fa
        from ._native import lib
        fa._call(lib().femgpu_halo_check(self.halo, C.c_void_p(stream)))

    def cg(self, b, x0=None, rtol: float = 1e-10, maxiter: int = 1000, check_every: int = 10, params=None):
        """Distributed CG on the devices (femgpu_halo_cg): dots over owned rows all-reduced GPU to GPU.
        b, x0: float64 CUDA tensors in the local test numbering.  Returns (x, iterations, rel residual)."""
        import torch

        from . import action as fa
        from ._native import lib
        x = torch.zeros_like(b) if x0 is None else x0.clone()
        torch.cuda.current_stream().synchronize()  # b and x are written before the instance stream reads them
        it, rel = C.c_int32(), C.c_double()
        # the ranks' common schedule: an automatic-schedule pass here would load modules (which may
        # wait for the device) while a peer already spins on this rank
        sp = fa._sched(params if params is not None else self.params)
        fa._call(lib().femgpu_halo_cg(self.halo, sp[0] if sp else None, C.c_void_p(b.data_ptr()),
                                      C.c_void_p(x.data_ptr()), rtol, maxiter, check_every, C.byref(it), C.byref(rel)))
        return x, it.value, rel.value

    def owned_output(self) -> Tuple[np.ndarray, np.ndarray]:
        """(global rows, values) of the rows this rank owns (complete after an action)."""
        y = self.inst.read_output()
        m = self.plan.owned_mask
        return self.plan.test_global[m], y[m]

    def close(self):
        from ._native import lib
        if self.halo:
            lib().femgpu_halo_destroy(self.halo)
            self.halo = None
        self.inst.close()


# ------------------------------------------------------------------------------- host emulation


def host_exchange(buf, send: Dict[int, np.ndarray], recv: Dict[int, np.ndarray], add: bool):
    """Point-to-point exchange of torch CPU tensors over torch.distributed (gloo): send buf[send[q]]
    to q, receive into buf[recv[q]], adding in ascending rank order when add=True."""
    import torch
    import torch.distributed as tdist
    ops, got = [], []
    for q in sorted(set(send) | set(recv)):
        if q in send:
            ops.append(tdist.P2POp(tdist.isend, buf[torch.as_tensor(send[q])].contiguous(), q))
        if q in recv:
            t = torch.empty(len(recv[q]), dtype=buf.dtype)
            got.append((q, t))
            ops.append(tdist.P2POp(tdist.irecv, t, q))
    if ops:
        for w in tdist.batch_isend_irecv(ops):
            w.wait()
    for q, t in sorted(got, key=lambda x: x[0]):
        idx = torch.as_tensor(recv[q])
        if add:
            buf.index_add_(0, idx, t)
        else:
            buf[idx] = t
    return buf


def host_halo_action(plan: RankPlan, local_apply, xs: Optional[List[np.ndarray]] = None) -> np.ndarray:
    """The distributed action with the plan's exchanges on the host (gloo) and the local compute
    by local_apply(problem) -> y: pull of ghost trial nodes from their owners (every space, vector
    spaces node-wise), local action, push of partial rows to the owners, owners add in ascending
    rank order.  xs: this rank's local trial inputs (owned values current; ghosts refreshed here)."""
    import torch
    p = plan.local
    xs = [np.array(x, dtype=np.float64) for x in (xs if xs is not None else list(p.scalar_inputs) + list(p.vector_inputs))]
    d = p.signature.dim
    ns = len(p.scalar_inputs)
    for s, x in enumerate(xs):
        comps = 1 if s < ns else d
        t = torch.as_tensor(x.reshape(-1, comps).copy())
        recv = {q: mine for q, (mine, _) in plan.pull[s].items()}
        for c in range(comps):
            col = t[:, c].contiguous()
            host_exchange(col, plan.serve[s], recv, False)
            t[:, c] = col
        xs[s] = t.numpy().reshape(-1).copy()
    q = ProblemInstance(p.signature, p.map, p.tabulations, p.connectivity, xs[:ns], xs[ns:], p.output_size)
    y = torch.as_tensor(np.asarray(local_apply(q), dtype=np.float64).copy())
    host_exchange(y, plan.push, plan.recv, True)
    return y.numpy()


def rank_slab(name_or_args, rank: int, world: int, n: Optional[int] = None) -> Slab:
    if isinstance(name_or_args, str):
        return config_slab(name_or_args, rank, world, n=n)
    form, dim, degree, Q, nn = name_or_args
    from .mesh import mesh_counts
    cells = mesh_counts(dim, nn, degree)[0]
    b, e = split_cells(cells, world, group_align(dim))[rank]
    return slab_instance(form, dim, degree, Q, nn, b, e)


def cpu_action_with_halo(name_or_args, rank: int, world: int, action, n: Optional[int] = None):
    """CPU leg for the gloo tests: this rank's slab, the collective plan and the host exchange with
    `action` (the oracle) as local compute; returns (owned global rows, owned y)."""
    plan = build_plan(rank_slab(name_or_args, rank, world, n), rank, world, torch_gather())
    y = host_halo_action(plan, action)
    m = plan.owned_mask
    return plan.test_global[m], y[m]


# ------------------------------------------------------------------------------- bench leg


def bench(args):
    """Multi-GPU bench leg (one process per GPU): strong scaling of the action on the fixed mesh,
    each rank building only its slab, halos GPU to GPU; max over ranks of the CUDA-event step time;
    rank 0 checks the gathered owned rows against the reference CPU action."""
    import torch
    import torch.distributed as tdist

    from . import action as fa
    from ._native import lib
    from .mesh import CONFIGS, mesh_counts

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, fa.device_count())
    device = local_rank % ndev
    tdist.init_process_group("gloo")  # control plane only; the data path is csrc/halo.cu
    gather = torch_gather()
    lib().femgpu_set_device(device)
    torch.cuda.set_device(device)
    t0 = time.perf_counter()
    slab = config_slab(args.config, rank, world, n=args.n)
    plan = build_plan(slab, rank, world, gather)
    t_plan = time.perf_counter() - t0
    di = DistInstance(plan, gather)
    tdist.barrier()
    for _ in range(max(args.warmup, 3)):
        di.action()
    di.check()
    # ---- timed region: exactly K distributed actions per rank (one CUDA graph launch each), CUDA
    # events on the rank's stream, barrier + device synchronize on both sides, max over ranks
    torch.cuda.synchronize()
    tdist.barrier()
    t_rank = di.time_steps(args.steps) / args.steps
    torch.cuda.synchronize()
    tdist.barrier()
    di.check()
    t = torch.tensor([t_rank], dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    t_step = float(t.item())
    launches = di.inst.stats()["launches_last_action"]
    gids, ys = di.owned_output()
    # ---- e2e through the public API with host buffers: each rank uploads its slab's inputs
    # (femgpu_set_inputs), runs the distributed action, downloads its output (femgpu_read_output)
    p = plan.local
    xs_h = [np.ascontiguousarray(x) for x in p.scalar_inputs]
    vs_h = [np.ascontiguousarray(x) for x in p.vector_inputs]
    h2d = sum(x.nbytes for x in xs_h + vs_h)
    d2h = 8 * p.output_size
    e2e_steps = max(2, min(args.e2e_steps, 20))
    tdist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        di.inst.set_inputs(xs_h, vs_h)
        di.action()
        di.inst.read_output()
    tdist.barrier()
    te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64)
    tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
    io = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64)
    tdist.all_reduce(io)
    di.check()
    parts = gather((gids, ys))
    stats = gather({"rank": rank, "device": device, "cells": int(plan.local.connectivity.cell_count),
                    "boundary_cells": plan.boundary_cells, "halo_rows": plan.halo_rows(),
                    "pull_nodes": int(sum(len(m) for d in plan.pull for m, _ in d.values())),
                    "step_us": t_rank * 1e6, "plan_s": round(t_plan, 2),
                    "schedule": di.inst.describe(di.params).split(" | auto: ")[0]})
    if rank == 0:
        c = dict(CONFIGS[args.config])
        if args.n is not None:
            c["n"] = args.n
        cells = mesh_counts(c["dim"], c["n"], c["degree"])[0]
        dofs = sum(len(g) for g, _ in parts)
        out = {
            "metric": "FP64 operator-action GDOF/s", "value": dofs / t_step / 1e9, "unit": "GDOF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s cell-partitioned over %d ranks (contiguous brick-major slabs, each rank builds "
                                   "only its own); per step: ghost inputs pulled from their owners, boundary cells, "
                                   "partial rows pushed to their owners over NVLink (CUDA IPC / peer pointers, "
                                   "device-side flags) overlapping the interior cells, owned rows completed in "
                                   "ascending rank order" % (args.config, world),
                       "cells": int(cells), "dofs": int(dofs), "parallelism": "cells%d" % world,
                       "devices_visible": ndev, "control_plane": "torch.distributed gloo (plan + handle exchange)"},
            "gpu_launches": args.steps * max(1, launches) * world,
            "e2e": {"value": dofs / float(te.item()) / 1e9, "unit": "GDOF/s", "h2d_bytes_per_step": int(io[0].item()),
                    "d2h_bytes_per_step": int(io[1].item()), "ms_per_step": float(te.item()) * 1e3,
                    "api": "per rank femgpu_set_inputs + femgpu_halo_action + femgpu_read_output (host buffers), "
                           "wall clock, max over ranks"},
            "ranks": stats,
        }
        y = np.full(dofs, np.nan)
        for g, v in parts:
            y[g] = v
        out["parity_complete"] = bool(not np.isnan(y).any())
        if not args.no_cpu_baseline:
            from . import mesh as fm
            p = fm.config_problem(args.config, n=args.n)
            try:
                from oracle import oracle  # the checker (reference build) on rank 0
                if oracle.ref_available():
                    _, ref = oracle.ref_time_threads(p, max(1, min(os.cpu_count() or 1, 64)), reps=1)
                    kind = "oracle/_ref reference_action, full workload"
                else:
                    ref = oracle.reference_action(p)
                    kind = "C restatement (oracle/femoracle.c), full workload"
                rel = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
                mx = float(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1e-30)))
                out["parity_vs_reference"] = {"rel_l2": rel, "max_rel": mx, "reference": kind,
                                              "pass": bool(rel <= 1e-12 and mx <= 1e-10)}
            except Exception as e:  # noqa: BLE001
                out["parity_vs_reference"] = {"error": str(e)[:200]}
        print(json.dumps(out), flush=True)
    tdist.barrier()
    di.close()
    tdist.destroy_process_group()
