// reorder.cpp — locality-restoring renumbering of a general mesh (femgpu_problem_reorder).
//
// The action's gathers and red.add scatter are fast when consecutive cells touch nearby index
// ranges: then a warp's loads share L1/L2 lines and the resident working set stays small.  A
// mesh numbered without locality (tools/general_mesh.py "global": C2 with shuffled cells, 1657 us
// per step instead of 370) is made local again here, once, on the host:
//   * cells are sorted by the Morton code of their centroid (affine geometry; otherwise by their
//     smallest node index), ties by the old cell index;
//   * every global index space is renumbered in first-touch order over the sorted cells (nodes no
//     cell touches keep their relative order at the end).  Spaces with the same global count share
//     one numbering, so a square operator's x and y stay in one numbering (Krylov loops); a vector
//     test space whose rows are node * dim + comp of a vector trial space follows that space's nodes.
// The result is the same problem in the new numbering: inputs and coordinates permuted, maps
// relabelled; its action is the old one permuted (y_new[r] = y_old[output_perm[r]]), up to the
// floating-point order of the per-row sums.
#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <vector>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}

uint64_t spread2(uint64_t v) {  // 32 bits -> every second bit
    v &= 0xffffffffULL;
    v = (v | v << 16) & 0x0000ffff0000ffffULL;
    v = (v | v << 8) & 0x00ff00ff00ff00ffULL;
    v = (v | v << 4) & 0x0f0f0f0f0f0f0f0fULL;
    v = (v | v << 2) & 0x3333333333333333ULL;
    v = (v | v << 1) & 0x5555555555555555ULL;
    return v;
}

// First-touch numbering of one index space over the sorted cells: perm[new] = old.
struct Numbering {
    std::vector<int32_t> old_of_new, new_of_old;
};

}  // namespace

femgpu_owned_problem* reorder_problem(const femgpu_problem* p, int32_t* cell_perm, int32_t* output_perm,
                                      int32_t* const* scalar_perms, int32_t* const* vector_perms) {
    validate_problem(p);
    const long long C = p->cell_count;
    const int d = p->dim;
    // ---- cell order
    std::vector<uint64_t> key(static_cast<size_t>(C));
    if (p->affine_geometry) {
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (long long v = 0; v < p->coord_global_count; ++v)
            for (int a = 0; a < d; ++a) {
                lo[a] = std::min(lo[a], p->coords[v * d + a]);
                hi[a] = std::max(hi[a], p->coords[v * d + a]);
            }
        const double bins = d == 3 ? 2097151.0 : d == 2 ? 4294967295.0 : 1.8e19;
        parallel_for(C, [&](long long b, long long e) {
            for (long long c = b; c < e; ++c) {
                uint64_t q[3] = {0, 0, 0};
                for (int a = 0; a < d; ++a) {
                    double s = 0.0;
                    for (int j = 0; j < p->coord_dofs; ++j) s += p->coords[static_cast<long long>(p->coord_map[c * p->coord_dofs + j]) * d + a];
                    const double t = hi[a] > lo[a] ? (s / p->coord_dofs - lo[a]) / (hi[a] - lo[a]) : 0.0;
                    q[a] = static_cast<uint64_t>(std::min(bins, std::max(0.0, t * bins)));
                }
                key[c] = d == 3 ? spread3(q[0]) | spread3(q[1]) << 1 | spread3(q[2]) << 2
                                : d == 2 ? spread2(q[0]) | spread2(q[1]) << 1 : q[0];
            }
        });
    } else if (p->n_scalar + p->n_vector > 0) {
        const femgpu_space& s = p->n_scalar ? p->scalar_spaces[0] : p->vector_spaces[0];
        for (long long c = 0; c < C; ++c) {
            int32_t m = INT32_MAX;
            for (int j = 0; j < s.dofs; ++j) m = std::min(m, s.map[c * s.dofs + j]);
            key[c] = static_cast<uint64_t>(m);
        }
    }
    std::vector<int32_t> order(static_cast<size_t>(C));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
    if (cell_perm) std::memcpy(cell_perm, order.data(), sizeof(int32_t) * static_cast<size_t>(C));
    // ---- index spaces: one numbering per global count, built from the first map with that count
    std::map<long long, Numbering> spaces;
    auto number = [&](const int32_t* map, int E, long long global) -> const Numbering& {
        auto it = spaces.find(global);
        if (it != spaces.end()) return it->second;
        Numbering n;
        n.new_of_old.assign(static_cast<size_t>(global), -1);
        n.old_of_new.reserve(static_cast<size_t>(global));
        for (long long k = 0; k < C; ++k) {
            const int32_t* row = map + static_cast<long long>(order[k]) * E;
            for (int j = 0; j < E; ++j)
                if (n.new_of_old[row[j]] < 0) {
                    n.new_of_old[row[j]] = static_cast<int32_t>(n.old_of_new.size());
                    n.old_of_new.push_back(row[j]);
                }
        }
        for (long long v = 0; v < global; ++v)
            if (n.new_of_old[v] < 0) {
                n.new_of_old[v] = static_cast<int32_t>(n.old_of_new.size());
                n.old_of_new.push_back(static_cast<int32_t>(v));
            }
        return spaces.emplace(global, std::move(n)).first->second;
    };
    // the vector test space convention (row = node * dim + comp of a vector trial space): its rows
    // follow that space's node numbering
    int tvec = -1;
    for (int i = 0; i < p->n_vector && tvec < 0; ++i) {
        const femgpu_space& s = p->vector_spaces[i];
        if (static_cast<long long>(s.dofs) * d != p->test_dofs || static_cast<long long>(s.global_count) * d != p->test_global_count) continue;
        bool ok = true;
        for (long long c = 0; c < C && ok; ++c)
            for (int a = 0; a < s.dofs && ok; ++a)
                for (int comp = 0; comp < d && ok; ++comp)
                    ok = p->test_map[c * p->test_dofs + a * d + comp] == s.map[c * s.dofs + a] * d + comp;
        if (ok) tvec = i;
    }
    // trial spaces first (so a square operator's test space shares the trial numbering)
    for (int i = 0; i < p->n_scalar; ++i) number(p->scalar_spaces[i].map, p->scalar_spaces[i].dofs, p->scalar_spaces[i].global_count);
    for (int i = 0; i < p->n_vector; ++i) number(p->vector_spaces[i].map, p->vector_spaces[i].dofs, p->vector_spaces[i].global_count);
    if (p->affine_geometry) number(p->coord_map, p->coord_dofs, p->coord_global_count);
    std::vector<int32_t> test_new_of_old;  // only for the vector test convention
    if (tvec >= 0) {
        const Numbering& n = spaces.at(p->vector_spaces[tvec].global_count);
        test_new_of_old.resize(static_cast<size_t>(p->test_global_count));
        for (long long v = 0; v < p->vector_spaces[tvec].global_count; ++v)
            for (int comp = 0; comp < d; ++comp) test_new_of_old[v * d + comp] = n.new_of_old[v] * d + comp;
    } else {
        test_new_of_old = number(p->test_map, p->test_dofs, p->test_global_count).new_of_old;
    }
    // ---- the renumbered problem
    auto P = std::make_unique<femgpu_owned_problem>();
    femgpu_problem& f = P->desc;
    f = *p;
    auto relabel = [&](const int32_t* map, int E, const std::vector<int32_t>& new_of_old) {
        std::vector<int32_t> out(static_cast<size_t>(C) * E);
        parallel_for(C, [&](long long b, long long e) {
            for (long long k = b; k < e; ++k)
                for (int j = 0; j < E; ++j) out[k * E + j] = new_of_old[map[static_cast<long long>(order[k]) * E + j]];
        });
        return out;
    };
    auto permute_rows = [&](const double* in, long long rows, int width, const std::vector<int32_t>& old_of_new) {
        std::vector<double> out(static_cast<size_t>(rows) * width);
        for (long long r = 0; r < rows; ++r)
            std::memcpy(&out[r * width], in + static_cast<long long>(old_of_new[r]) * width, sizeof(double) * width);
        return out;
    };
    P->sspaces.assign(p->scalar_spaces, p->scalar_spaces + p->n_scalar);
    P->vspaces.assign(p->vector_spaces, p->vector_spaces + p->n_vector);
    for (int i = 0; i < p->n_scalar; ++i) {
        const femgpu_space& s = p->scalar_spaces[i];
        const Numbering& n = spaces.at(s.global_count);
        P->smaps.push_back(relabel(s.map, s.dofs, n.new_of_old));
        P->sin.push_back(permute_rows(s.input, s.global_count, 1, n.old_of_new));
        P->sphi.emplace_back(s.phi, s.phi + static_cast<size_t>(s.deriv_terms) * p->quad_points * s.dofs);
        if (scalar_perms && scalar_perms[i]) std::memcpy(scalar_perms[i], n.old_of_new.data(), sizeof(int32_t) * s.global_count);
    }
    for (int i = 0; i < p->n_vector; ++i) {
        const femgpu_space& s = p->vector_spaces[i];
        const Numbering& n = spaces.at(s.global_count);
        P->vmaps.push_back(relabel(s.map, s.dofs, n.new_of_old));
        P->vin.push_back(permute_rows(s.input, s.global_count, d, n.old_of_new));
        P->vphi.emplace_back(s.phi, s.phi + static_cast<size_t>(s.deriv_terms) * p->quad_points * s.dofs);
        P->comps.emplace_back(s.components, s.components + s.deriv_terms);
        if (vector_perms && vector_perms[i]) std::memcpy(vector_perms[i], n.old_of_new.data(), sizeof(int32_t) * s.global_count);
    }
    P->test_map = relabel(p->test_map, p->test_dofs, test_new_of_old);
    if (output_perm) {
        for (long long v = 0; v < p->test_global_count; ++v) output_perm[test_new_of_old[v]] = static_cast<int32_t>(v);
    }
    if (p->affine_geometry) {
        const Numbering& n = spaces.at(p->coord_global_count);
        P->coord_map = relabel(p->coord_map, p->coord_dofs, n.new_of_old);
        P->coords = permute_rows(p->coords, p->coord_global_count, d, n.old_of_new);
    }
    P->psi.assign(p->psi, p->psi + static_cast<size_t>(p->test_deriv_terms) * p->test_dofs * p->quad_points);
    P->weights.assign(p->weights, p->weights + p->quad_points);
    P->nodes.assign(p->map_nodes, p->map_nodes + p->n_map_nodes);
    P->outputs.assign(p->map_outputs, p->map_outputs + p->n_map_outputs);
    for (size_t i = 0; i < P->sspaces.size(); ++i) {
        P->sspaces[i].phi = P->sphi[i].data();
        P->sspaces[i].map = P->smaps[i].data();
        P->sspaces[i].input = P->sin[i].data();
        P->sspaces[i].components = nullptr;
    }
    for (size_t i = 0; i < P->vspaces.size(); ++i) {
        P->vspaces[i].phi = P->vphi[i].data();
        P->vspaces[i].map = P->vmaps[i].data();
        P->vspaces[i].input = P->vin[i].data();
        P->vspaces[i].components = P->comps[i].data();
    }
    f.scalar_spaces = P->sspaces.empty() ? nullptr : P->sspaces.data();
    f.vector_spaces = P->vspaces.empty() ? nullptr : P->vspaces.data();
    f.psi = P->psi.data();
    f.weights = P->weights.data();
    f.test_map = P->test_map.data();
    f.coord_map = f.affine_geometry ? P->coord_map.data() : nullptr;
    f.coords = f.affine_geometry ? P->coords.data() : nullptr;
    f.map_nodes = P->nodes.data();
    f.map_outputs = P->outputs.data();
    validate_problem(&f);
    return P.release();
}

}  // namespace femgpu

extern "C" femgpu_status femgpu_problem_reorder(const femgpu_problem* p, femgpu_owned_problem** out, const femgpu_problem** view,
                                                int32_t* cell_perm, int32_t* output_perm, int32_t* const* scalar_input_perms,
                                                int32_t* const* vector_input_perms) {
    return femgpu::abi_guard([&] {
        if (!p || !out || !view) femgpu::invalid("reorder: null argument");
        femgpu_owned_problem* P = femgpu::reorder_problem(p, cell_perm, output_perm, scalar_input_perms, vector_input_perms);
        *out = P;
        *view = &P->desc;
    });
}
