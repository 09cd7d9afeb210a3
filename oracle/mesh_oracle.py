"""TEST INFRASTRUCTURE ONLY — independent pure-Python restatement of the structured mesh
generator (femgpu_mesh_build, paper_2506_17471_b200/csrc/mesh.cpp) used to pin its cell-node
maps, vertex maps and coordinates bit-exactly, and of the greedy colouring
(femgpu_color_cells).  The reference has no mesh generator (its instances are chain-connected,
form.hpp:759-768); these meshes are inputs to the same ProblemInstance data model.

Conventions (must match mesh.cpp): vertex v = i + (n+1) j [+ (n+1)^2 l], coordinates lattice/n;
cells brick-major (bricks of brick^d squares/cubes, lexicographic; squares/cubes lexicographic
within a brick); square -> triangles (v00, v10, v11), (v00, v11, v01); cube -> 6 Kuhn tetrahedra
along the axis permutations in lexicographic order, odd permutations with the last two vertices
swapped (positive orientation); P_k nodes: the d+1 vertices first, then the remaining
barycentric multi-indices in lexicographic order of (a_1..a_d); node id = lattice index on the
(k n + 1)^d lattice of sum_i a_i V_i.
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
    return verts + rest


def _simplices(d, i, j, l):
    if d == 2:
        c = [(i, j), (i + 1, j), (i + 1, j + 1), (i, j + 1)]
        return [[c[0], c[1], c[2]], [c[0], c[2], c[3]]]
    out = []
    for perm in itertools.permutations(range(3)):
        p = [i, j, l]
        path = [tuple(p)]
        for ax in perm:
            p[ax] += 1
            path.append(tuple(p))
        inversions = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b])
        if inversions % 2:
            path[2], path[3] = path[3], path[2]
        out.append(path)
    return out


def mesh(d, n, k, brick):
    lat = _lattice(d, k)
    kn1 = k * n + 1
    nb = (n + brick - 1) // brick
    node_map, vert_map = [], []
    zr = range(nb) if d == 3 else range(1)
    for bz in zr:
        for by in range(nb):
            for bx in range(nb):
                ls = range(bz * brick, min(n, bz * brick + brick)) if d == 3 else range(1)
                for l in ls:
                    for j in range(by * brick, min(n, by * brick + brick)):
                        for i in range(bx * brick, min(n, bx * brick + brick)):
                            for V in _simplices(d, i, j, l):
                                vrow = []
                                for v in V:
                                    idx = v[0] + (n + 1) * v[1] + ((n + 1) ** 2 * v[2] if d == 3 else 0)
                                    vrow.append(idx)
                                vert_map.append(vrow)
                                nrow = []
                                for a in lat:
                                    pnt = [sum(a[t] * V[t][c] for t in range(d + 1)) for c in range(d)]
                                    nrow.append(pnt[0] + kn1 * pnt[1] + (kn1 * kn1 * pnt[2] if d == 3 else 0))
                                node_map.append(nrow)
    nv = (n + 1) ** d
    coords = np.zeros((nv, d))
    for v in range(nv):
        coords[v, 0] = (v % (n + 1)) / n
        coords[v, 1] = ((v // (n + 1)) % (n + 1)) / n
        if d == 3:
            coords[v, 2] = (v // ((n + 1) ** 2)) / n
    return np.array(node_map, dtype=np.int32), np.array(vert_map, dtype=np.int32), coords


def greedy_colors(m):
    colors = []
    adj = {}
    for row in m:
        forbidden = set()
        for g in row:
            forbidden |= adj.get(int(g), set())
        c = 0
        while c in forbidden:
            c += 1
        colors.append(c)
        for g in row:
            adj.setdefault(int(g), set()).add(c)
    return np.array(colors, dtype=np.int32)
