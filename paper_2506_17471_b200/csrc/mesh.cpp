// mesh.cpp — synthetic structured simplex meshes (unit square / unit cube) and a
// deterministic greedy cell colouring.  The reference has no mesh generator
// (its instances are chain-connected, form.hpp:759-768); these feed the same
// ProblemInstance data model so the oracle runs on identical meshes.
//
// Layout choices (B200-first): cells are emitted brick-major, i.e. bricks of
// brick^d squares/cubes in lexicographic order and the squares/cubes of one brick
// in lexicographic order, so a run of consecutive cells (one CTA tile) is
// spatially compact and its DOFs are largely private to it.
#include <algorithm>
#include <array>
#include <cstdint>
#include <vector>

#include "femgpu_internal.hpp"

namespace {

// Barycentric multi-indices of P_k on a d-simplex: vertices first (k*e_i), then the
// rest in lexicographic order of (a_1, ..., a_d).
std::vector<std::array<int, 4>> lattice_nodes(int d, int k) {
    std::vector<std::array<int, 4>> verts, rest;
    for (int i = 0; i <= d; ++i) {
        std::array<int, 4> a{0, 0, 0, 0};
        a[i] = k;
        verts.push_back(a);
    }
    auto is_vertex = [&](const std::array<int, 4>& a) {
        for (int i = 0; i <= d; ++i)
            if (a[i] == k) return true;
        return false;
    };
    std::array<int, 4> a{0, 0, 0, 0};
    if (d == 1) {
        for (int a1 = 0; a1 <= k; ++a1) {
            a = {k - a1, a1, 0, 0};
            if (!is_vertex(a)) rest.push_back(a);
        }
    } else if (d == 2) {
        for (int a1 = 0; a1 <= k; ++a1)
            for (int a2 = 0; a1 + a2 <= k; ++a2) {
                a = {k - a1 - a2, a1, a2, 0};
                if (!is_vertex(a)) rest.push_back(a);
            }
    } else {
        for (int a1 = 0; a1 <= k; ++a1)
            for (int a2 = 0; a1 + a2 <= k; ++a2)
                for (int a3 = 0; a1 + a2 + a3 <= k; ++a3) {
                    a = {k - a1 - a2 - a3, a1, a2, a3};
                    if (!is_vertex(a)) rest.push_back(a);
                }
    }
    verts.insert(verts.end(), rest.begin(), rest.end());
    return verts;
}

// Cell vertices (integer lattice coordinates in [0, n]) for square/cube (i, j, l), local simplex s.
void simplex_vertices(int d, int i, int j, int l, int s, int V[4][3]) {
    if (d == 2) {
        const int c[4][2] = {{i, j}, {i + 1, j}, {i + 1, j + 1}, {i, j + 1}};
        const int tri[2][3] = {{0, 1, 2}, {0, 2, 3}};
        for (int v = 0; v < 3; ++v) {
            V[v][0] = c[tri[s][v]][0];
            V[v][1] = c[tri[s][v]][1];
            V[v][2] = 0;
        }
        return;
    }
    // Kuhn tetrahedra: monotone lattice path from (0,0,0) to (1,1,1) along permutation pi;
    // odd permutations swap the last two vertices so every tetrahedron is positively oriented.
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const bool odd[6] = {false, true, true, false, false, true};
    int p[3] = {i, j, l};
    for (int v = 0; v < 3; ++v) V[0][v] = p[v];
    for (int step = 0; step < 3; ++step) {
        p[perms[s][step]] += 1;
        for (int v = 0; v < 3; ++v) V[step + 1][v] = p[v];
    }
    if (odd[s])
        for (int v = 0; v < 3; ++v) std::swap(V[2][v], V[3][v]);
}

}  // namespace

extern "C" {

femgpu_status femgpu_mesh_counts(int32_t dim, int32_t n, int32_t degree, int64_t* cells, int64_t* nodes,
                                 int64_t* vertices, int32_t* nodes_per_cell) {
    if (dim < 2 || dim > 3 || n < 1 || degree < 1 || degree > 8) return FEMGPU_E_INVALID;
    const int64_t sc = dim == 2 ? 2 : 6;
    int64_t c = sc, nn = 1, vv = 1;
    for (int i = 0; i < dim; ++i) {
        c *= n;
        nn *= static_cast<int64_t>(degree) * n + 1;
        vv *= n + 1;
    }
    if (c > INT32_MAX || nn > INT32_MAX) return FEMGPU_E_INVALID;
    if (cells) *cells = c;
    if (nodes) *nodes = nn;
    if (vertices) *vertices = vv;
    if (nodes_per_cell) {
        int npc = 1;
        for (int i = 1; i <= dim; ++i) npc = npc * (degree + i) / i;
        // binomial(degree+dim, dim) computed incrementally is exact for these sizes
        *nodes_per_cell = npc;
    }
    return FEMGPU_OK;
}

femgpu_status femgpu_mesh_build(int32_t dim, int32_t n, int32_t degree, int32_t brick, int32_t* node_map,
                                int32_t* vertex_map, double* coords) {
    int64_t cells = 0;
    if (femgpu_mesh_counts(dim, n, degree, &cells, nullptr, nullptr, nullptr) != FEMGPU_OK) return FEMGPU_E_INVALID;
    return femgpu_mesh_build_range(dim, n, degree, brick, 0, cells, node_map, vertex_map, coords);
}

femgpu_status femgpu_mesh_build_range(int32_t dim, int32_t n, int32_t degree, int32_t brick, int64_t cell_begin,
                                      int64_t cell_end, int32_t* node_map, int32_t* vertex_map, double* coords) {
    int64_t cells = 0, nodes = 0, verts = 0;
    int32_t npc = 0;
    if (femgpu_mesh_counts(dim, n, degree, &cells, &nodes, &verts, &npc) != FEMGPU_OK) return FEMGPU_E_INVALID;
    if (cell_begin < 0 || cell_end < cell_begin || cell_end > cells) return FEMGPU_E_INVALID;
    if (brick < 1) brick = 1;
    const auto lat = lattice_nodes(dim, degree);
    if (static_cast<int>(lat.size()) != npc) return FEMGPU_E_INTERNAL;
    const int sc = dim == 2 ? 2 : 6;
    const int64_t kn1 = static_cast<int64_t>(degree) * n + 1;
    const int nb = (n + brick - 1) / brick;
    int64_t cell = 0;
    int V[4][3];
    const int nbz = dim == 3 ? nb : 1;
    for (int bz = 0; bz < nbz; ++bz)
        for (int by = 0; by < nb; ++by)
            for (int bx = 0; bx < nb; ++bx) {
                const int z0 = bz * brick, z1 = dim == 3 ? std::min(n, z0 + brick) : 1;
                const int y0 = by * brick, y1 = std::min(n, y0 + brick);
                const int x0 = bx * brick, x1 = std::min(n, x0 + brick);
                const int64_t brick_cells = static_cast<int64_t>(z1 - (dim == 3 ? z0 : 0)) * (y1 - y0) * (x1 - x0) * sc;
                if (cell + brick_cells <= cell_begin || cell >= cell_end) {  // brick outside the range
                    cell += brick_cells;
                    continue;
                }
                for (int l = (dim == 3 ? z0 : 0); l < z1; ++l)
                    for (int j = y0; j < y1; ++j)
                        for (int i = x0; i < x1; ++i)
                            for (int s = 0; s < sc; ++s, ++cell) {
                                if (cell < cell_begin || cell >= cell_end) continue;
                                const int64_t out = cell - cell_begin;  // row in the caller's arrays
                                simplex_vertices(dim, i, j, l, s, V);
                                if (vertex_map)
                                    for (int v = 0; v <= dim; ++v) {
                                        int64_t idx = V[v][0] + static_cast<int64_t>(n + 1) * V[v][1];
                                        if (dim == 3) idx += static_cast<int64_t>(n + 1) * (n + 1) * V[v][2];
                                        vertex_map[out * (dim + 1) + v] = static_cast<int32_t>(idx);
                                    }
                                if (node_map)
                                    for (int a = 0; a < npc; ++a) {
                                        int64_t p[3] = {0, 0, 0};
                                        for (int v = 0; v <= dim; ++v)
                                            for (int c = 0; c < dim; ++c) p[c] += static_cast<int64_t>(lat[a][v]) * V[v][c];
                                        int64_t idx = p[0] + kn1 * p[1];
                                        if (dim == 3) idx += kn1 * kn1 * p[2];
                                        node_map[out * npc + a] = static_cast<int32_t>(idx);
                                    }
                            }
            }
    if (coords) {
        const int64_t n1 = n + 1;
        for (int64_t v = 0; v < verts; ++v) {
            const int64_t i = v % n1, j = (v / n1) % n1, l = v / (n1 * n1);
            coords[v * dim + 0] = static_cast<double>(i) / n;
            coords[v * dim + 1] = static_cast<double>(j) / n;
            if (dim == 3) coords[v * dim + 2] = static_cast<double>(l) / n;
        }
    }
    return FEMGPU_OK;
}

femgpu_status femgpu_color_cells(const int32_t* map, int32_t cells, int32_t entries, int32_t global_count,
                                 int32_t* colors, int32_t* n_colors) {
    if (!map || !colors || cells < 1 || entries < 1 || global_count < 1) return FEMGPU_E_INVALID;
    // used[g] = bitmask of colours already adjacent to entry g (up to 64 colours per word).
    std::vector<std::vector<uint64_t>> used(1, std::vector<uint64_t>(static_cast<size_t>(global_count), 0));
    int nc = 0;
    for (int64_t c = 0; c < cells; ++c) {
        int color = -1;
        for (size_t w = 0; color < 0; ++w) {
            if (w == used.size()) used.emplace_back(static_cast<size_t>(global_count), 0);
            uint64_t forbidden = 0;
            for (int j = 0; j < entries; ++j) forbidden |= used[w][map[c * entries + j]];
            if (~forbidden) color = static_cast<int>(w * 64 + __builtin_ctzll(~forbidden));
        }
        colors[c] = color;
        for (int j = 0; j < entries; ++j) used[color / 64][map[c * entries + j]] |= 1ULL << (color % 64);
        nc = std::max(nc, color + 1);
    }
    if (n_colors) *n_colors = nc;
    return FEMGPU_OK;
}

}  // extern "C"
