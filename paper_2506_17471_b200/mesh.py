"""Synthetic refined unit-square / unit-cube problems for the benchmark configs.

Meshes come from libfemgpu's native generator (femgpu_mesh_build, mesh.cpp):
P_k nodes on the k-refined lattice, global DOF = lattice index, cells ordered
brick-major.  Tabulations, weights and inputs use the reference's synthesis
distributions (SynthRng, make_problem, form.hpp:774-852) and seed.  The same
ProblemInstance feeds both the GPU path and the CPU oracle, so both see
identical meshes and inputs.

Forms (BASELINE.json configs):
  mass / laplace / helmholtz / elasticity / hyperelasticity   reference presets (form.hpp:625-734)
  helmholtz_coef   P_k Helmholtz with a P1 coefficient field kappa on the vertex map (C3)
  advection        (b . grad u, v) with a P1 vector velocity b; uses w*adj(J) (= w*det*J^-1),
                   expressible in the reference map language (C5)
  hyperelastic     St. Venant-Kirchhoff tangent around a P_k coefficient displacement u0
                   (nonlinear, coefficient-dependent; C5)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from ._native import check, lib
from .form import (FormSignature, IndexMap, MeshConnectivity, PointwiseMap, ProblemInstance, ScalarSpace,
                   SynthRng, Tabulations, VectorSpace, _draw_tabulations, _metric_entry, _seed0, preset_map,
                   preset_signature, simplex_space_dim)

FORMS = ("mass", "laplace", "helmholtz", "elasticity", "hyperelasticity", "helmholtz_coef", "advection",
         "hyperelastic")


def default_brick(dim: int) -> int:
    return 4 if dim == 3 else 8


def mesh_counts(dim: int, n: int, degree: int):
    cells, nodes, verts, npc = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
    check(lib().femgpu_mesh_counts(dim, n, degree, C.byref(cells), C.byref(nodes), C.byref(verts), C.byref(npc)))
    return cells.value, nodes.value, verts.value, npc.value


def unit_mesh(dim: int, n: int, degree: int, brick: int | None = None):
    """(node_map [cells, npc], vertex_map [cells, dim+1], coords [verts, dim], n_nodes, n_verts)."""
    brick = default_brick(dim) if brick is None else brick
    cells, nodes, verts, npc = mesh_counts(dim, n, degree)
    node_map = np.empty((cells, npc), dtype=np.int32)
    vertex_map = np.empty((cells, dim + 1), dtype=np.int32)
    coords = np.empty((verts, dim), dtype=np.float64)
    check(lib().femgpu_mesh_build(dim, n, degree, brick, abi.iptr(node_map), abi.iptr(vertex_map), abi.dptr(coords)))
    return node_map, vertex_map, coords, nodes, verts


def color_cells(map_: np.ndarray, global_count: int):
    cells, entries = map_.shape
    colors = np.empty(cells, dtype=np.int32)
    nc = C.c_int32()
    m = np.ascontiguousarray(map_, dtype=np.int32)
    check(lib().femgpu_color_cells(abi.iptr(m), cells, entries, global_count, abi.iptr(colors), C.byref(nc)))
    return colors, nc.value


# --------------------------------------------------------------------------- extra forms


def _adjugate(m: PointwiseMap, d: int):
    """adj(J)[r][c] nodes (adj(J) = det(J) J^-1) using add/mul/constant only."""
    J = lambda r, c: m.jacobian(r, c)  # noqa: E731
    if d == 2:
        return [[J(1, 1), m.mul(m.constant(-1.0), J(0, 1))], [m.mul(m.constant(-1.0), J(1, 0)), J(0, 0)]]
    adj = [[None] * 3 for _ in range(3)]
    for r in range(3):
        for c in range(3):
            # adj[r][c] = cofactor[c][r] = (-1)^(r+c) * minor(c, r)
            rows = [i for i in range(3) if i != c]
            cols = [j for j in range(3) if j != r]
            minor = m.sub(m.mul(J(rows[0], cols[0]), J(rows[1], cols[1])), m.mul(J(rows[0], cols[1]), J(rows[1], cols[0])))
            adj[r][c] = minor if (r + c) % 2 == 0 else m.mul(m.constant(-1.0), minor)
    return adj


def form_signature(form: str, dim: int, degree: int, Q: int) -> FormSignature:
    if form in ("mass", "laplace", "poisson", "helmholtz", "elasticity", "hyperelasticity"):
        return preset_signature(form, dim, degree, Q)
    n = simplex_space_dim(degree, dim)
    sig = FormSignature(dim=dim, quad_points=Q, coord_dofs=dim + 1, affine_geometry=True, word_bytes=8)
    if form == "helmholtz_coef":
        sig.scalar_spaces = [ScalarSpace(n, dim + 1), ScalarSpace(dim + 1, 1)]
        sig.test_dofs, sig.test_deriv_terms = n, dim + 1
    elif form == "advection":
        sig.scalar_spaces = [ScalarSpace(n, dim)]
        sig.vector_spaces = [VectorSpace(dim + 1, dim, list(range(dim)))]
        sig.test_dofs, sig.test_deriv_terms = n, 1
    elif form == "hyperelastic":
        comps = [a for a in range(dim) for _c in range(dim)]
        sig.vector_spaces = [VectorSpace(n, dim * dim, comps), VectorSpace(n, dim * dim, list(comps))]
        sig.test_dofs, sig.test_deriv_terms = n * dim, dim * dim
    else:
        raise ValueError("unknown form: " + form)
    sig.validate()
    return sig


def form_map(form: str, sig: FormSignature) -> PointwiseMap:
    if form in ("mass", "laplace", "poisson", "helmholtz", "elasticity", "hyperelasticity"):
        return preset_map(form, sig)
    d = sig.dim
    m = PointwiseMap()
    if form == "helmholtz_coef":
        wd = m.mul(m.weight(), m.determinant())
        for r in range(d):
            terms = [m.mul(_metric_entry(m, d, r, c), m.scalar_deriv(0, c)) for c in range(d)]
            m.add_output(m.mul(wd, m.sum(terms)))
        m.add_output(m.mul(wd, m.mul(m.scalar_deriv(1, 0), m.scalar_deriv(0, d))))
    elif form == "advection":
        # w*det*(b . J^-T grad_ref u) = w * sum_c (sum_r adj(J)[c][r] b_r) d_c u
        adj = _adjugate(m, d)
        w = m.weight()
        terms = []
        for c in range(d):
            bc = m.sum([m.mul(adj[c][r], m.vector_deriv(0, r)) for r in range(d)])
            terms.append(m.mul(bc, m.scalar_deriv(0, c)))
        m.add_output(m.mul(w, m.sum(terms)))
    elif form == "hyperelastic":
        # St. Venant-Kirchhoff tangent dP = dF S + F dS around F = I + grad(u0), written with the
        # symmetry of C = F^T F and dE = (M + M^T)/2, M = dF^T F (the same form as the textbook
        # E = (C - I)/2, S = 2 mu E + lam tr(E) I, dS = 2 mu dE + lam tr(dE) I, in ~30 % fewer map ops):
        #   S = mu (C - I) + lam/2 (tr C - d) I,   dS = mu (M + M^T) + lam tr(M) I
        lam, mu = 1.25, 0.75
        wd = m.mul(m.weight(), m.determinant())
        dF = [[m.vector_deriv(0, a * d + c) for c in range(d)] for a in range(d)]          # grad(du)
        G0 = [[m.vector_deriv(1, a * d + c) for c in range(d)] for a in range(d)]          # grad(u0)
        F = [[m.add(m.constant(1.0), G0[a][c]) if a == c else G0[a][c] for c in range(d)] for a in range(d)]
        C = {}
        for a in range(d):
            for c in range(a, d):
                C[a, c] = C[c, a] = m.sum([m.mul(F[k][a], F[k][c]) for k in range(d)])
        M = [[m.sum([m.mul(dF[k][a], F[k][c]) for k in range(d)]) for c in range(d)] for a in range(d)]
        trC = m.sum([C[k, k] for k in range(d)])
        trM = m.sum([M[k][k] for k in range(d)])
        muc = m.constant(mu)
        s0 = m.add(m.mul(m.constant(0.5 * lam), trC), m.constant(-mu - 0.5 * lam * d))
        ltrM = m.mul(m.constant(lam), trM)
        S, dS = {}, {}
        for a in range(d):
            for c in range(a, d):
                S[a, c] = S[c, a] = m.add(m.mul(muc, C[a, c]), s0) if a == c else m.mul(muc, C[a, c])
                dS[a, c] = dS[c, a] = (m.add(m.mul(m.constant(2.0 * mu), M[a][a]), ltrM) if a == c
                                       else m.mul(muc, m.add(M[a][c], M[c][a])))
        for a in range(d):
            for c in range(d):
                dP = m.add(m.sum([m.mul(dF[a][k], S[k, c]) for k in range(d)]),
                           m.sum([m.mul(F[a][k], dS[k, c]) for k in range(d)]))
                m.add_output(m.mul(wd, dP))
    else:
        raise ValueError("unknown form: " + form)
    m.validate(sig)
    return m


def mesh_problem(form: str, dim: int, degree: int, Q: int, n: int, seed: int = 7, brick: int | None = None,
                 scale_u0: float = 0.05, mesh=None) -> ProblemInstance:
    """A ProblemInstance on the structured unit mesh with make_problem's data distributions.
    `mesh` = (node_map, vertex_map, coords) supplies the mesh arrays instead of the native
    generator (the reference arm of bench.py builds them without loading libfemgpu)."""
    sig = form_signature(form, dim, degree, Q)
    pmap = form_map(form, sig)
    if mesh is None:
        node_map, vertex_map, coords, n_nodes, n_verts = unit_mesh(dim, n, degree, brick)
    else:
        node_map, vertex_map, coords = mesh
        n_nodes, n_verts = (degree * n + 1) ** dim, (n + 1) ** dim
    rng = SynthRng(_seed0(seed))
    tab = _draw_tabulations(sig, rng)
    cells = node_map.shape[0]
    conn = MeshConnectivity(cell_count=cells)
    nodes_im = IndexMap(node_map, int(n_nodes))
    verts_im = IndexMap(vertex_map, int(n_verts))
    npc = node_map.shape[1]
    for s in sig.scalar_spaces:
        conn.scalar_maps.append(nodes_im if s.dofs == npc else verts_im)
    for v in sig.vector_spaces:
        conn.vector_maps.append(nodes_im if v.dofs == npc else verts_im)
    if sig.test_dofs == npc:
        conn.test_map = nodes_im
    else:  # vector test space, node-major local order j = a*d + c
        d = dim
        tm = (node_map[:, :, None].astype(np.int64) * d + np.arange(d)[None, None, :]).reshape(cells, npc * d)
        conn.test_map = IndexMap(tm.astype(np.int32), int(n_nodes) * d)
    conn.coord_map = verts_im
    conn.coords = coords
    conn.coord_global_count = int(n_verts)
    p = ProblemInstance(sig, pmap, tab, conn)
    for mm in conn.scalar_maps:
        p.scalar_inputs.append(rng.uniform(0.25, 1.0, mm.global_count))
    for i, mm in enumerate(conn.vector_maps):
        x = rng.uniform(0.25, 1.0, mm.global_count * dim)
        if form == "hyperelastic" and i == 1:
            x = x * scale_u0  # coefficient displacement: a small deformation
        p.vector_inputs.append(x)
    p.output_size = conn.test_map.global_count
    p.validate()
    return p


# Benchmark configurations (BASELINE.json configs; Q and N per SURVEY §8d).
CONFIGS = {
    "C1": dict(form="mass", dim=2, degree=1, Q=3, n=256),
    "C1b": dict(form="mass", dim=2, degree=1, Q=3, n=4096),
    "C2": dict(form="laplace", dim=3, degree=2, Q=4, n=107),
    "C3a": dict(form="helmholtz_coef", dim=2, degree=3, Q=12, n=1024),
    "C3b": dict(form="helmholtz_coef", dim=3, degree=3, Q=24, n=48),
    "C4": dict(form="elasticity", dim=3, degree=2, Q=4, n=128),
    "C5-adv-P1": dict(form="advection", dim=3, degree=1, Q=4, n=256),
    "C5-adv-P2": dict(form="advection", dim=3, degree=2, Q=14, n=128),
    "C5-adv-P3": dict(form="advection", dim=3, degree=3, Q=24, n=85),
    "C5-adv-P4": dict(form="advection", dim=3, degree=4, Q=46, n=64),
    "C5-hyp-P1": dict(form="hyperelastic", dim=3, degree=1, Q=4, n=160),
    "C5-hyp-P2": dict(form="hyperelastic", dim=3, degree=2, Q=14, n=80),
    "C5-hyp-P3": dict(form="hyperelastic", dim=3, degree=3, Q=24, n=56),
    "C5-hyp-P4": dict(form="hyperelastic", dim=3, degree=4, Q=46, n=40),
}


def config_problem(name: str, n: int | None = None, seed: int = 7, mesh_fn=None) -> ProblemInstance:
    """Benchmark configuration `name`; mesh_fn(dim, n, degree, brick) -> (node_map, vertex_map,
    coords) replaces the native mesh generator."""
    c = dict(CONFIGS[name])
    if n is not None:
        c["n"] = n
    mesh = mesh_fn(c["dim"], c["n"], c["degree"], default_brick(c["dim"])) if mesh_fn else None
    return mesh_problem(c["form"], c["dim"], c["degree"], c["Q"], c["n"], seed=seed, mesh=mesh)


# Fused-action pairs (fuse.py): operators that share their trial function on one mesh.
FUSED_PAIRS = {
    # velocity block and divergence constraint of a Stokes-type system on P2 velocities (C4's mesh):
    # both read the P2 vector field u; the divergence terms are 3 of the velocity block's 9 gradients
    "stokes-P2": dict(dim=3, degree=2, Q=4, n=128),
    # stiffness and mass on the same P2 scalar field (C2's mesh; the operators of M + dt K)
    "laplace+mass-P2": dict(dim=3, degree=2, Q=4, n=107),
}


def fused_pair(name: str, n: int | None = None, seed: int = 7):
    """(A, B): two problems on one mesh, quadrature and trial vector (the operands of fuse_problems)."""
    c = dict(FUSED_PAIRS[name])
    if n is not None:
        c["n"] = n
    d, deg, Q, nn = c["dim"], c["degree"], c["Q"], c["n"]
    if name.startswith("laplace+mass"):
        a = mesh_problem("laplace", d, deg, Q, nn, seed=seed)
        b = mesh_problem("mass", d, deg, Q, nn, seed=seed + 1)
        b.tabulations.weights = a.tabulations.weights.copy()
        b.scalar_inputs = [x.copy() for x in a.scalar_inputs]
        return a, b
    a = mesh_problem("elasticity", d, deg, Q, nn, seed=seed)
    # divergence: trial = a's vector space restricted to the terms d_a u_a (a's term a*d + a, component
    # a, same tabulation rows), test = P1 scalar on the vertices, w det (sum_a d_a u_a)
    sig = FormSignature(dim=d, quad_points=Q, coord_dofs=d + 1, affine_geometry=True, word_bytes=8)
    npc = a.signature.vector_spaces[0].dofs
    sig.vector_spaces = [VectorSpace(npc, d, list(range(d)))]
    sig.test_dofs, sig.test_deriv_terms = d + 1, 1
    sig.validate()
    m = PointwiseMap()
    wd = m.mul(m.weight(), m.determinant())
    m.add_output(m.mul(wd, m.sum([m.vector_deriv(0, k) for k in range(d)])))
    m.validate(sig)
    rng = SynthRng(_seed0(seed + 1))
    tab = Tabulations()
    tab.vector_phi = [np.ascontiguousarray(a.tabulations.vector_phi[0][[k * d + k for k in range(d)]])]
    tab.psi = np.asarray(rng.uniform(0.1, 1.1, (d + 1) * Q)).reshape(1, d + 1, Q)
    tab.weights = a.tabulations.weights.copy()
    ca = a.connectivity
    conn = MeshConnectivity(cell_count=ca.cell_count, vector_maps=[ca.vector_maps[0]], test_map=ca.coord_map,
                            coord_map=ca.coord_map, coords=ca.coords, coord_global_count=ca.coord_global_count)
    b = ProblemInstance(sig, m, tab, conn, [], [a.vector_inputs[0].copy()], ca.coord_map.global_count)
    b.validate()
    return a, b
