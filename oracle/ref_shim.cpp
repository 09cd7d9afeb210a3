// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  Compiles the UNMODIFIED reference
// header (/root/reference/proj/include/femsched/form.hpp, included in place via
// -I, never copied) into oracle/_ref/libfemsched_ref.so, and exposes it through
// a small extern "C" surface so the Python tests and bench.py's CPU baseline
// can run the reference's own code:
//
//   ref_reference_action  -> femsched::reference_action            form.hpp:471-595
//   ref_make_preset       -> femsched::preset_signature/preset_map  form.hpp:625-734
//                            + make_problem / generic_map           form.hpp:774-881
//   ref_usable_flops      -> femsched::usable_flops                 form.hpp:164-173
//   ref_time_threads      -> the reference action on T host threads over contiguous
//                            cell ranges (restriction of test_form.cpp:11-24),
//                            outputs summed in rank order.
//
// Build recipe: oracle/Makefile (outputs only into oracle/_ref/).
#include <femsched/form.hpp>
#include <femsched/io.hpp>  // needs boost/rational.hpp: third_party/boost shim (qoi.hpp)

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../include/femgpu.h"

using namespace femsched;

namespace {

int set_err(char* err, int len, const std::string& msg) {
    if (err && len > 0) {
        std::strncpy(err, msg.c_str(), static_cast<std::size_t>(len) - 1);
        err[len - 1] = 0;
    }
    return 0;
}

IndexMap to_map(const int32_t* m, int cells, int entries, int global) {
    IndexMap out(cells, entries, global);
    std::memcpy(out.indices.data(), m, sizeof(int) * static_cast<std::size_t>(cells) * entries);
    return out;
}

// Builds a femsched::ProblemInstance from the flat descriptor.
ProblemInstance from_desc(const femgpu_problem* d, int cell_begin, int cell_end) {
    ProblemInstance p;
    FormSignature& s = p.signature;
    s.dim = d->dim;
    s.quad_points = d->quad_points;
    s.coord_dofs = d->coord_dofs;
    s.affine_geometry = d->affine_geometry != 0;
    s.coordinate_space = d->coordinate_space;
    s.word_bytes = d->word_bytes;
    s.test_dofs = d->test_dofs;
    s.test_deriv_terms = d->test_deriv_terms;
    const int Q = d->quad_points;
    const int cells = cell_end - cell_begin;
    auto mat = [](const double* src, int rows, int cols) {
        Matrix m(rows, cols);
        std::memcpy(m.data.data(), src, sizeof(double) * static_cast<std::size_t>(rows) * cols);
        return m;
    };
    p.tabulations.scalar_phi.resize(d->n_scalar);
    p.tabulations.vector_phi.resize(d->n_vector);
    p.connectivity.cell_count = cells;
    for (int i = 0; i < d->n_scalar; ++i) {
        const femgpu_space& sp = d->scalar_spaces[i];
        s.scalar_spaces.push_back({sp.dofs, sp.deriv_terms});
        for (int k = 0; k < sp.deriv_terms; ++k)
            p.tabulations.scalar_phi[i].push_back(mat(sp.phi + static_cast<std::size_t>(k) * Q * sp.dofs, Q, sp.dofs));
        p.connectivity.scalar_maps.push_back(
            to_map(sp.map + static_cast<std::size_t>(cell_begin) * sp.dofs, cells, sp.dofs, sp.global_count));
        p.scalar_inputs.emplace_back(sp.input, sp.input + sp.global_count);
    }
    for (int i = 0; i < d->n_vector; ++i) {
        const femgpu_space& sp = d->vector_spaces[i];
        VectorSpace v;
        v.dofs = sp.dofs;
        v.deriv_terms = sp.deriv_terms;
        v.components.assign(sp.components, sp.components + sp.deriv_terms);
        s.vector_spaces.push_back(v);
        for (int k = 0; k < sp.deriv_terms; ++k)
            p.tabulations.vector_phi[i].push_back(mat(sp.phi + static_cast<std::size_t>(k) * Q * sp.dofs, Q, sp.dofs));
        p.connectivity.vector_maps.push_back(
            to_map(sp.map + static_cast<std::size_t>(cell_begin) * sp.dofs, cells, sp.dofs, sp.global_count));
        p.vector_inputs.emplace_back(sp.input, sp.input + static_cast<std::size_t>(sp.global_count) * d->dim);
    }
    for (int k = 0; k < d->test_deriv_terms; ++k)
        p.tabulations.psi.push_back(mat(d->psi + static_cast<std::size_t>(k) * d->test_dofs * Q, d->test_dofs, Q));
    p.tabulations.weights.assign(d->weights, d->weights + Q);
    p.connectivity.test_map = to_map(d->test_map + static_cast<std::size_t>(cell_begin) * d->test_dofs, cells,
                                     d->test_dofs, d->test_global_count);
    if (s.affine_geometry) {
        p.connectivity.coord_map = to_map(d->coord_map + static_cast<std::size_t>(cell_begin) * d->coord_dofs,
                                          cells, d->coord_dofs, d->coord_global_count);
        p.connectivity.coord_global_count = d->coord_global_count;
        p.connectivity.coords.assign(d->coords,
                                     d->coords + static_cast<std::size_t>(d->coord_global_count) * d->dim);
    }
    // Rebuild the map through the public builder so node ids are identical.
    PointwiseMap& m = p.map;
    for (int id = 0; id < d->n_map_nodes; ++id) {
        const femgpu_map_node& n = d->map_nodes[id];
        switch (n.op) {
            case FEMGPU_OP_CONSTANT: m.constant(n.value); break;
            case FEMGPU_OP_SCALAR_DERIV: m.scalar_deriv(n.a, n.b); break;
            case FEMGPU_OP_VECTOR_DERIV: m.vector_deriv(n.a, n.b); break;
            case FEMGPU_OP_JACOBIAN: m.jacobian(n.a, n.b); break;
            case FEMGPU_OP_DETERMINANT: m.determinant(); break;
            case FEMGPU_OP_WEIGHT: m.weight(); break;
            case FEMGPU_OP_COORD: m.coord(n.a, n.b); break;
            case FEMGPU_OP_ADD: m.add(n.a, n.b); break;
            case FEMGPU_OP_MUL: m.mul(n.a, n.b); break;
            default: throw std::invalid_argument("ref_shim: map op not expressible in the reference");
        }
    }
    for (int o = 0; o < d->n_map_outputs; ++o) m.add_output(d->map_outputs[o]);
    p.output_size = d->output_size;
    return p;
}

// Compact restriction of cells [b, e): every map is renumbered to the indices the range
// touches (ascending), inputs/coords are gathered accordingly, and test_global (the local->
// global test numbering) is returned so partial outputs can be summed into the global y.
ProblemInstance compact_from_desc(const femgpu_problem* d, int b, int e, std::vector<int>& test_global) {
    ProblemInstance p = from_desc(d, b, e);  // global numbering, restricted maps
    auto compact = [](IndexMap& m, std::vector<int>& uniq) {
        uniq.assign(m.indices.begin(), m.indices.end());
        std::sort(uniq.begin(), uniq.end());
        uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
        for (int& v : m.indices) v = static_cast<int>(std::lower_bound(uniq.begin(), uniq.end(), v) - uniq.begin());
        m.global_count = static_cast<int>(uniq.size());
    };
    std::vector<int> u;
    for (std::size_t i = 0; i < p.connectivity.scalar_maps.size(); ++i) {
        compact(p.connectivity.scalar_maps[i], u);
        std::vector<double> x(u.size());
        for (std::size_t k = 0; k < u.size(); ++k) x[k] = p.scalar_inputs[i][u[k]];
        p.scalar_inputs[i] = std::move(x);
    }
    const int dim = p.signature.dim;
    for (std::size_t i = 0; i < p.connectivity.vector_maps.size(); ++i) {
        compact(p.connectivity.vector_maps[i], u);
        std::vector<double> x(u.size() * dim);
        for (std::size_t k = 0; k < u.size(); ++k)
            for (int c = 0; c < dim; ++c) x[k * dim + c] = p.vector_inputs[i][static_cast<std::size_t>(u[k]) * dim + c];
        p.vector_inputs[i] = std::move(x);
    }
    if (p.signature.affine_geometry) {
        compact(p.connectivity.coord_map, u);
        std::vector<double> X(u.size() * dim);
        for (std::size_t k = 0; k < u.size(); ++k)
            for (int c = 0; c < dim; ++c) X[k * dim + c] = p.connectivity.coords[static_cast<std::size_t>(u[k]) * dim + c];
        p.connectivity.coords = std::move(X);
        p.connectivity.coord_global_count = static_cast<int>(u.size());
    }
    compact(p.connectivity.test_map, test_global);
    p.output_size = p.connectivity.test_map.global_count;
    return p;
}

// Owns a reference-generated instance and a flat descriptor pointing into it.
struct Held {
    ProblemInstance p;
    std::vector<std::vector<double>> phi_flat;
    std::vector<std::vector<int>> comps;
    std::vector<double> psi_flat;
    std::vector<femgpu_space> scalar, vector;
    std::vector<femgpu_map_node> nodes;
    std::vector<int> outputs;
    femgpu_problem desc{};
};

void flatten(Held& h) {
    const ProblemInstance& p = h.p;
    const FormSignature& s = p.signature;
    const int Q = s.quad_points;
    auto flat = [](const std::vector<Matrix>& ms) {
        std::vector<double> out;
        for (const auto& m : ms) out.insert(out.end(), m.data.begin(), m.data.end());
        return out;
    };
    for (std::size_t i = 0; i < s.scalar_spaces.size(); ++i) h.phi_flat.push_back(flat(p.tabulations.scalar_phi[i]));
    for (std::size_t i = 0; i < s.vector_spaces.size(); ++i) {
        h.phi_flat.push_back(flat(p.tabulations.vector_phi[i]));
        h.comps.push_back(s.vector_spaces[i].components);
    }
    h.psi_flat = flat(p.tabulations.psi);
    std::size_t f = 0;
    for (std::size_t i = 0; i < s.scalar_spaces.size(); ++i, ++f) {
        femgpu_space sp{};
        sp.dofs = s.scalar_spaces[i].dofs;
        sp.deriv_terms = s.scalar_spaces[i].deriv_terms;
        sp.phi = h.phi_flat[f].data();
        sp.map = p.connectivity.scalar_maps[i].indices.data();
        sp.global_count = p.connectivity.scalar_maps[i].global_count;
        sp.input = p.scalar_inputs[i].data();
        h.scalar.push_back(sp);
    }
    for (std::size_t i = 0; i < s.vector_spaces.size(); ++i, ++f) {
        femgpu_space sp{};
        sp.dofs = s.vector_spaces[i].dofs;
        sp.deriv_terms = s.vector_spaces[i].deriv_terms;
        sp.components = h.comps[i].data();
        sp.phi = h.phi_flat[f].data();
        sp.map = p.connectivity.vector_maps[i].indices.data();
        sp.global_count = p.connectivity.vector_maps[i].global_count;
        sp.input = p.vector_inputs[i].data();
        h.vector.push_back(sp);
    }
    for (const auto& n : p.map.nodes()) {
        femgpu_map_node o{};
        o.op = static_cast<int32_t>(n.op);
        o.a = n.a;
        o.b = n.b;
        o.value = n.value;
        h.nodes.push_back(o);
    }
    h.outputs = p.map.outputs();
    femgpu_problem& d = h.desc;
    d.dim = s.dim;
    d.quad_points = Q;
    d.coord_dofs = s.coord_dofs;
    d.affine_geometry = s.affine_geometry;
    d.coordinate_space = s.coordinate_space;
    d.word_bytes = s.word_bytes;
    d.n_scalar = static_cast<int32_t>(h.scalar.size());
    d.n_vector = static_cast<int32_t>(h.vector.size());
    d.scalar_spaces = h.scalar.data();
    d.vector_spaces = h.vector.data();
    d.test_dofs = s.test_dofs;
    d.test_deriv_terms = s.test_deriv_terms;
    d.psi = h.psi_flat.data();
    d.weights = p.tabulations.weights.data();
    d.cell_count = p.connectivity.cell_count;
    d.test_global_count = p.connectivity.test_map.global_count;
    d.test_map = p.connectivity.test_map.indices.data();
    d.coord_map = s.affine_geometry ? p.connectivity.coord_map.indices.data() : nullptr;
    d.coords = s.affine_geometry ? p.connectivity.coords.data() : nullptr;
    d.coord_global_count = p.connectivity.coord_global_count;
    d.n_map_nodes = static_cast<int32_t>(h.nodes.size());
    d.map_nodes = h.nodes.data();
    d.map_outputs = h.outputs.data();
    d.n_map_outputs = static_cast<int32_t>(h.outputs.size());
    d.output_size = p.output_size;
}

}  // namespace

extern "C" {

// 0 ok, 1 invalid_argument, 3 runtime_error (non-finite), 6 other
int ref_reference_action(const femgpu_problem* d, double* out, long long* counters, char* err, int len) {
    try {
        ProblemInstance p = from_desc(d, 0, d->cell_count);
        ReferenceCounters c;
        auto y = reference_action(p, counters ? &c : nullptr);
        std::memcpy(out, y.data(), sizeof(double) * y.size());
        if (counters) {
            counters[0] = c.matvec_mults;
            counters[1] = c.matvec_adds;
            counters[2] = c.map_ops;
        }
        return 0;
    } catch (const std::invalid_argument& e) {
        set_err(err, len, e.what());
        return 1;
    } catch (const std::runtime_error& e) {
        set_err(err, len, e.what());
        return 3;
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return 6;
    }
}

// op: mass|laplace|poisson|helmholtz|elasticity|hyperelasticity, or "generic:<preset>"
// for the preset signature with generic_map.  Returns nullptr on error.
void* ref_make_preset(const char* op, int dim, int degree, int quad_points, int cells, unsigned long long seed,
                      char* err, int len) {
    try {
        std::string name(op);
        bool generic = false;
        if (name.rfind("generic:", 0) == 0) {
            generic = true;
            name = name.substr(8);
        }
        const Operator o = operator_from_name(name);
        const FormSignature sig = preset_signature(o, dim, degree, quad_points);
        auto h = std::make_unique<Held>();
        h->p = generic ? make_problem(sig, generic_map(sig), cells, seed)
                       : make_problem(sig, preset_map(o, sig), cells, seed);
        flatten(*h);
        return h.release();
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return nullptr;
    }
}

const femgpu_problem* ref_instance_desc(void* h) { return &static_cast<Held*>(h)->desc; }

void ref_free(void* h) { delete static_cast<Held*>(h); }

long long ref_usable_flops(const char* op, int dim, int degree, int quad_points) {
    try {
        return usable_flops(preset_signature(operator_from_name(op), dim, degree, quad_points));
    } catch (const std::exception&) {
        return -1;
    }
}

// CPU baseline harness: T threads, each running the unmodified reference_action on a
// compact sub-instance of a contiguous cell range (domain decomposition); the partial
// outputs are summed into out in rank order.  Timing excludes sub-instance construction
// and includes the summation.  Returns mean seconds per action, < 0 on error.
double ref_time_threads(const femgpu_problem* d, int cell_begin, int cell_end, int threads, int reps,
                        double* out, char* err, int len) {
    try {
        if (threads < 1) threads = 1;
        const int cells = cell_end - cell_begin;
        if (threads > cells) threads = cells;
        std::vector<ProblemInstance> parts(threads);
        std::vector<std::vector<int>> tg(threads);
        {
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; ++t)
                pool.emplace_back([&, t] {
                    const int b = cell_begin + static_cast<int>(static_cast<long long>(cells) * t / threads);
                    const int e = cell_begin + static_cast<int>(static_cast<long long>(cells) * (t + 1) / threads);
                    parts[t] = compact_from_desc(d, b, e, tg[t]);
                });
            for (auto& th : pool) th.join();
        }
        std::vector<std::vector<double>> ys(threads);
        std::vector<double> y(static_cast<std::size_t>(d->output_size), 0.0);
        double total = 0.0;
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; ++t)
                pool.emplace_back([&, t] { ys[t] = reference_action(parts[t]); });
            for (auto& th : pool) th.join();
            std::fill(y.begin(), y.end(), 0.0);
            for (int t = 0; t < threads; ++t)
                for (std::size_t i = 0; i < tg[t].size(); ++i) y[tg[t][i]] += ys[t][i];
            const auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
        }
        if (out) std::memcpy(out, y.data(), sizeof(double) * y.size());
        return total / reps;
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return -1.0;
    }
}

// femsched::save_instance_file / load_instance_file (io.hpp:381-391), for the io parity tests.
int ref_save_instance(const femgpu_problem* d, const char* path, char* err, int len) {
    try {
        femsched::save_instance_file(path, from_desc(d, 0, d->cell_count));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return 1;
    }
}

void* ref_load_instance(const char* path, char* err, int len) {
    try {
        auto h = std::make_unique<Held>();
        h->p = femsched::load_instance_file(path);
        flatten(*h);
        return h.release();
    } catch (const std::exception& e) {
        set_err(err, len, e.what());
        return nullptr;
    }
}

}  // extern "C"
