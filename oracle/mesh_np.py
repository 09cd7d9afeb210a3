"""TEST INFRASTRUCTURE ONLY — vectorised numpy restatement of the structured mesh generator
(femgpu_mesh_build, paper_2506_17471_b200/csrc/mesh.cpp), used where the checker must not load the
product library: the reference arm of bench.py builds its meshes with it, so that process runs
only the reference's own code (oracle/_ref) and this file.  Pinned bit-exact against the
pure-Python loops of oracle/mesh_oracle.py (small meshes) and against libfemgpu (benchmark
meshes) by tests/test_native_cpu.py.

Conventions (mesh_oracle.py docstring): brick-major cells (bricks of brick^d squares/cubes in
lexicographic order, squares/cubes lexicographic inside a brick); square -> 2 triangles, cube ->
6 positively oriented Kuhn tetrahedra; P_k node id = lattice index on the (k n + 1)^d lattice.
"""
import itertools

import numpy as np


def _lattice(d, k):
    verts = []
    for i in range(d + 1):
        a = [0] * (d + 1)
        a[i] = k
        verts.append(tuple(a))
    rest = []
    for tail in itertools.product(range(k + 1), repeat=d):
        if sum(tail) <= k:
            a = (k - sum(tail),) + tail
            if k not in a:
                rest.append(a)
    return np.array(verts + rest, dtype=np.int64)  # [npc, d+1]


def _simplex_offsets(d):
    """[s, d+1 vertices, d] integer offsets of the simplices of the unit square/cube."""
    if d == 2:
        c = [(0, 0), (1, 0), (1, 1), (0, 1)]
        return np.array([[c[0], c[1], c[2]], [c[0], c[2], c[3]]], dtype=np.int64)
    out = []
    for perm in itertools.permutations(range(3)):
        p = [0, 0, 0]
        path = [tuple(p)]
        for ax in perm:
            p[ax] += 1
            path.append(tuple(p))
        inversions = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b])
        if inversions % 2:
            path[2], path[3] = path[3], path[2]
        out.append(path)
    return np.array(out, dtype=np.int64)


def _cube_order(d, n, brick):
    """Integer coordinates [cubes, d] of the squares/cubes in brick-major order."""
    ax = np.arange(n, dtype=np.int64)
    grids = np.meshgrid(*([ax] * d), indexing="ij")  # grids[0] = i (x) ... lexicographic with x fastest
    coords = [g.ravel() for g in grids]               # coords[c] for axis c
    nb = (n + brick - 1) // brick
    key = np.zeros(coords[0].size, dtype=np.int64)
    # bricks lexicographic (z, y, x), then cubes lexicographic (z, y, x) inside the brick
    for c in reversed(range(d)):
        key = key * nb + coords[c] // brick
    for c in reversed(range(d)):
        key = key * brick + coords[c] % brick
    order = np.argsort(key, kind="stable")
    return np.stack([x[order] for x in coords], axis=1)


def mesh(d, n, k, brick):
    """(node_map [cells, npc] int32, vertex_map [cells, d+1] int32, coords [verts, d] f64)."""
    lat = _lattice(d, k)
    off = _simplex_offsets(d)                      # [S, d+1, d]
    cube = _cube_order(d, n, brick)                # [C, d]
    S = off.shape[0]
    n1, kn1 = n + 1, k * n + 1
    vstride = np.array([n1 ** c for c in range(d)], dtype=np.int64)
    kstride = np.array([kn1 ** c for c in range(d)], dtype=np.int64)
    vbase = cube @ vstride                         # vertex id of the cube origin
    kbase = k * (cube @ kstride)                   # refined-lattice id of the cube origin
    voff = off @ vstride                           # [S, d+1]
    # node a of simplex s: sum_v lat[a, v] * (origin + off[s, v]) on the refined lattice
    noff = np.einsum("av,svc,c->sa", lat, off, kstride)  # [S, npc]
    vertex_map = (vbase[:, None, None] + voff[None, :, :]).reshape(-1, d + 1)
    node_map = (kbase[:, None, None] + noff[None, :, :]).reshape(-1, lat.shape[0])
    v = np.arange(n1 ** d, dtype=np.int64)
    coords = np.stack([((v // n1 ** c) % n1) / n for c in range(d)], axis=1)
    assert vertex_map.shape[0] == S * n ** d
    return node_map.astype(np.int32), vertex_map.astype(np.int32), coords.astype(np.float64)
