// fuse.cpp — fused multi-operator actions (the follow-on of PAPER.md:2477-2482: "action kernels
// sharing trial functions ... fused ... would reduce the number of memory accesses").
//
// m problems on the same cells, geometry and quadrature become ONE problem whose output is the
// concatenation [y_1; ...; y_m]:
//   * trial spaces with the same map, global count and input are merged into one space carrying the
//     union of their derivative terms (a term = its component and its tabulation rows, identical
//     terms shared), so every shared trial value is gathered and evaluated once per cell;
//   * the map DAGs are concatenated (derivative leaves re-pointed at the merged terms); the
//     emitters' value numbering (dedupe_map) then shares common subexpressions (w*det, J^T J, ...);
//   * the test space is the disjoint union: local test DOFs of problem p map to offset_p + its rows,
//     Psi is block diagonal over (problem's outputs) x (problem's test DOFs).
// The reference algorithm on the fused problem computes exactly y_1..y_m (the off-diagonal Psi
// blocks are zeros); the emitted kernels skip the FMAs of Psi entries that are zero at every
// quadrature point (Signature::psi_nz), so the fused quadrature stage costs what the separate ones
// cost, while the gathers, geometry and shared evaluations are paid once.
#include <climits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

bool same_bytes(const void* a, const void* b, size_t n) { return n == 0 || a == b || std::memcmp(a, b, n) == 0; }

// One merged trial space: its identity (map, global count, input) and its terms.
struct MergedSpace {
    int dofs = 0, global = 0;
    const int32_t* map = nullptr;
    const double* input = nullptr;
    std::vector<int> comps;                 // vector spaces: component per term
    std::vector<std::vector<double>> rows;  // per term: Q x dofs tabulation
};

int find_or_add_space(std::vector<MergedSpace>& ms, const femgpu_space& s, long long cells, long long in_len) {
    for (size_t i = 0; i < ms.size(); ++i) {
        const MergedSpace& m = ms[i];
        if (m.dofs == s.dofs && m.global == s.global_count &&
            same_bytes(m.map, s.map, sizeof(int32_t) * static_cast<size_t>(cells * s.dofs)) &&
            same_bytes(m.input, s.input, sizeof(double) * static_cast<size_t>(in_len)))
            return static_cast<int>(i);
    }
    MergedSpace m;
    m.dofs = s.dofs;
    m.global = s.global_count;
    m.map = s.map;
    m.input = s.input;
    ms.push_back(std::move(m));
    return static_cast<int>(ms.size() - 1);
}

int find_or_add_term(MergedSpace& m, int comp, const double* row, size_t n) {
    for (size_t t = 0; t < m.rows.size(); ++t)
        if ((m.comps.empty() || m.comps[t] == comp) && same_bytes(m.rows[t].data(), row, sizeof(double) * n))
            return static_cast<int>(t);
    m.rows.emplace_back(row, row + n);
    if (comp >= 0) m.comps.push_back(comp);
    return static_cast<int>(m.rows.size() - 1);
}

}  // namespace

femgpu_owned_problem* fuse_problems(const femgpu_problem* const* probs, int n, int64_t* offsets) {
    if (n < 1 || !probs) invalid("fuse: at least one problem required");
    for (int p = 0; p < n; ++p) {
        if (!probs[p]) invalid("fuse: null problem");
        validate_problem(probs[p]);
    }
    const femgpu_problem& a = *probs[0];
    const long long C = a.cell_count;
    const int Q = a.quad_points, d = a.dim;
    for (int p = 1; p < n; ++p) {
        const femgpu_problem& b = *probs[p];
        if (b.dim != d || b.quad_points != Q || b.cell_count != C || b.coord_dofs != a.coord_dofs ||
            b.affine_geometry != a.affine_geometry || b.word_bytes != a.word_bytes)
            invalid("fuse: problems differ in dimension, quadrature, cell count or geometry kind");
        if (!same_bytes(a.weights, b.weights, sizeof(double) * Q)) invalid("fuse: quadrature weights differ");
        if (a.affine_geometry) {
            if (b.coord_global_count != a.coord_global_count ||
                !same_bytes(a.coord_map, b.coord_map, sizeof(int32_t) * static_cast<size_t>(C * a.coord_dofs)) ||
                !same_bytes(a.coords, b.coords, sizeof(double) * static_cast<size_t>(a.coord_global_count) * d))
                invalid("fuse: problems differ in mesh geometry (coordinate map or coordinates)");
        }
    }
    auto P = std::make_unique<femgpu_owned_problem>();
    femgpu_problem& f = P->desc;
    f.dim = d;
    f.quad_points = Q;
    f.coord_dofs = a.coord_dofs;
    f.affine_geometry = a.affine_geometry;
    f.word_bytes = a.word_bytes;
    f.cell_count = a.cell_count;
    // ---- merged trial spaces and the term remapping of every problem
    std::vector<MergedSpace> ms_s, ms_v;
    // per problem: (space, term) -> (merged space, merged term)
    std::vector<std::vector<std::vector<std::pair<int, int>>>> smap(n), vmap(n);
    std::vector<int> coord_space(n, -1);
    for (int p = 0; p < n; ++p) {
        const femgpu_problem& b = *probs[p];
        smap[p].resize(b.n_scalar);
        for (int i = 0; i < b.n_scalar; ++i) {
            const femgpu_space& s = b.scalar_spaces[i];
            const int I = find_or_add_space(ms_s, s, C, s.global_count);
            for (int t = 0; t < s.deriv_terms; ++t)
                smap[p][i].push_back({I, find_or_add_term(ms_s[I], -1, s.phi + static_cast<size_t>(t) * Q * s.dofs,
                                                          static_cast<size_t>(Q) * s.dofs)});
        }
        vmap[p].resize(b.n_vector);
        for (int i = 0; i < b.n_vector; ++i) {
            const femgpu_space& s = b.vector_spaces[i];
            const int I = find_or_add_space(ms_v, s, C, static_cast<long long>(s.global_count) * d);
            for (int t = 0; t < s.deriv_terms; ++t)
                vmap[p][i].push_back({I, find_or_add_term(ms_v[I], s.components[t], s.phi + static_cast<size_t>(t) * Q * s.dofs,
                                                          static_cast<size_t>(Q) * s.dofs)});
            if (!b.affine_geometry && b.coordinate_space == i) coord_space[p] = I;
        }
    }
    if (!a.affine_geometry) {
        for (int p = 1; p < n; ++p)
            if (coord_space[p] != coord_space[0]) invalid("fuse: problems use different coordinate spaces");
        f.coordinate_space = coord_space[0];
    } else {
        f.coordinate_space = -1;
    }
    if (ms_s.size() > FEMGPU_MAX_SPACES || ms_v.size() > FEMGPU_MAX_SPACES) invalid("fuse: too many distinct trial spaces");
    auto emit_spaces = [&](std::vector<MergedSpace>& ms, bool vec) {
        auto& spaces = vec ? P->vspaces : P->sspaces;
        auto& phis = vec ? P->vphi : P->sphi;
        auto& maps = vec ? P->vmaps : P->smaps;
        auto& ins = vec ? P->vin : P->sin;
        for (MergedSpace& m : ms) {
            femgpu_space s{};
            s.dofs = m.dofs;
            s.deriv_terms = static_cast<int>(m.rows.size());
            s.global_count = m.global;
            spaces.push_back(s);
            std::vector<double> phi;
            for (const auto& r : m.rows) phi.insert(phi.end(), r.begin(), r.end());
            phis.push_back(std::move(phi));
            maps.emplace_back(m.map, m.map + C * m.dofs);
            const long long len = vec ? static_cast<long long>(m.global) * d : m.global;
            ins.emplace_back(m.input, m.input + len);
            if (vec) P->comps.push_back(m.comps);
        }
    };
    emit_spaces(ms_s, false);
    emit_spaces(ms_v, true);
    // ---- test space: disjoint union; Psi block diagonal
    int nW = 0, Tw = 0;
    long long rows = 0;
    std::vector<int> w_off(n), t_off(n);
    for (int p = 0; p < n; ++p) {
        w_off[p] = nW;
        t_off[p] = Tw;
        if (offsets) offsets[p] = rows;
        nW += probs[p]->test_dofs;
        Tw += probs[p]->test_deriv_terms;
        rows += probs[p]->output_size;
    }
    if (offsets) offsets[n] = rows;
    if (rows > INT32_MAX) invalid("fuse: fused output exceeds 2^31 rows");
    f.test_dofs = nW;
    f.test_deriv_terms = Tw;
    f.output_size = static_cast<int>(rows);
    f.test_global_count = static_cast<int>(rows);
    P->psi.assign(static_cast<size_t>(Tw) * nW * Q, 0.0);
    P->test_map.resize(static_cast<size_t>(C) * nW);
    long long row0 = 0;
    for (int p = 0; p < n; ++p) {
        const femgpu_problem& b = *probs[p];
        for (int k = 0; k < b.test_deriv_terms; ++k)
            for (int j = 0; j < b.test_dofs; ++j)
                std::memcpy(&P->psi[(static_cast<size_t>(t_off[p] + k) * nW + w_off[p] + j) * Q],
                            b.psi + (static_cast<size_t>(k) * b.test_dofs + j) * Q, sizeof(double) * Q);
        for (long long c = 0; c < C; ++c)
            for (int j = 0; j < b.test_dofs; ++j)
                P->test_map[static_cast<size_t>(c) * nW + w_off[p] + j] =
                    static_cast<int32_t>(row0 + b.test_map[static_cast<size_t>(c) * b.test_dofs + j]);
        row0 += b.output_size;
    }
    P->weights.assign(a.weights, a.weights + Q);
    if (a.affine_geometry) {
        P->coord_map.assign(a.coord_map, a.coord_map + C * a.coord_dofs);
        P->coords.assign(a.coords, a.coords + static_cast<size_t>(a.coord_global_count) * d);
        f.coord_global_count = a.coord_global_count;
    }
    // ---- map: concatenated DAGs, derivative leaves re-pointed, outputs in problem order
    for (int p = 0; p < n; ++p) {
        const femgpu_problem& b = *probs[p];
        const int base = static_cast<int>(P->nodes.size());
        for (int i = 0; i < b.n_map_nodes; ++i) {
            femgpu_map_node nd = b.map_nodes[i];
            if (nd.op == FEMGPU_OP_SCALAR_DERIV) {
                const auto st = smap[p][nd.a][nd.b];
                nd.a = st.first;
                nd.b = st.second;
            } else if (nd.op == FEMGPU_OP_VECTOR_DERIV) {
                const auto st = vmap[p][nd.a][nd.b];
                nd.a = st.first;
                nd.b = st.second;
            } else if (nd.op == FEMGPU_OP_ADD || nd.op == FEMGPU_OP_MUL) {
                nd.a += base;
                nd.b += base;
            }
            P->nodes.push_back(nd);
        }
        for (int k = 0; k < b.n_map_outputs; ++k) P->outputs.push_back(base + b.map_outputs[k]);
    }
    // ---- wire the descriptor to the owned storage
    for (size_t i = 0; i < P->sspaces.size(); ++i) {
        femgpu_space& s = P->sspaces[i];
        s.components = nullptr;
        s.phi = P->sphi[i].data();
        s.map = P->smaps[i].data();
        s.input = P->sin[i].data();
    }
    for (size_t i = 0; i < P->vspaces.size(); ++i) {
        femgpu_space& v = P->vspaces[i];
        v.components = P->comps[i].data();
        v.phi = P->vphi[i].data();
        v.map = P->vmaps[i].data();
        v.input = P->vin[i].data();
    }
    f.n_scalar = static_cast<int>(P->sspaces.size());
    f.n_vector = static_cast<int>(P->vspaces.size());
    f.scalar_spaces = P->sspaces.empty() ? nullptr : P->sspaces.data();
    f.vector_spaces = P->vspaces.empty() ? nullptr : P->vspaces.data();
    f.psi = P->psi.data();
    f.weights = P->weights.data();
    f.test_map = P->test_map.data();
    f.coord_map = f.affine_geometry ? P->coord_map.data() : nullptr;
    f.coords = f.affine_geometry ? P->coords.data() : nullptr;
    f.n_map_nodes = static_cast<int>(P->nodes.size());
    f.map_nodes = P->nodes.data();
    f.map_outputs = P->outputs.data();
    f.n_map_outputs = static_cast<int>(P->outputs.size());
    validate_problem(&f);
    return P.release();
}

}  // namespace femgpu

extern "C" femgpu_status femgpu_problem_fuse(const femgpu_problem* const* problems, int32_t n, femgpu_owned_problem** out,
                                             const femgpu_problem** view, int64_t* offsets) {
    return femgpu::abi_guard([&] {
        if (!out || !view) femgpu::invalid("fuse: null output handle");
        femgpu_owned_problem* P = femgpu::fuse_problems(problems, n, offsets);
        *out = P;
        *view = &P->desc;
    });
}
