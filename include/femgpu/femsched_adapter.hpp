// femsched_adapter.hpp — C++ drop-in for the reference's action path (header-only).
//
// A femsched user keeps their own headers (proj/include/femsched/*.hpp) and swaps
//
//     std::vector<double> y = femsched::reference_action(inst);          // form.hpp:471-472
//     auto res = femsched::tune(inst, dev, cfg, jobs);                    // search.hpp:338-339
// for
//     std::vector<double> y = femgpu::action(inst);                       // B200, same shape
//     auto res = femsched::tune(inst, dev, cfg, jobs, femgpu::executor()); // measuring Executor
//
// Everything crosses into libfemgpu through the C-ABI of <femgpu.h> (plain pointers, no
// exceptions).  Status codes come back as the reference's exception types:
//   FEMGPU_E_INVALID -> std::invalid_argument, FEMGPU_E_INFEASIBLE -> femsched::InfeasibleError,
//   FEMGPU_E_NONFINITE and others -> std::runtime_error (same "non-finite value at cell N during
//   <stage>" text as form.hpp:492-495).
// femgpu::executor() needs <femsched/search.hpp> (define FEMGPU_WITH_FEMSCHED_SEARCH first, or
// include search.hpp before this header).
#pragma once

#include <femsched/form.hpp>

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../femgpu.h"

#if defined(FEMGPU_WITH_FEMSCHED_SEARCH) || defined(FEMSCHED_SEARCH_HPP_INCLUDED)
#include <femsched/search.hpp>
#define FEMGPU_HAS_EXECUTOR 1
#endif

namespace femgpu {

inline void check(femgpu_status st) {
    if (st == FEMGPU_OK) return;
    const std::string msg = femgpu_last_error();
    if (st == FEMGPU_E_INVALID) throw std::invalid_argument(msg);
    if (st == FEMGPU_E_INFEASIBLE) throw femsched::InfeasibleError(msg);
    throw std::runtime_error(msg);
}

// Flat view of a femsched::ProblemInstance (borrowed pointers, valid while both live).
class ProblemView {
public:
    explicit ProblemView(const femsched::ProblemInstance& p) {
        const auto& sig = p.signature;
        const int Q = sig.quad_points;
        auto flat = [](const std::vector<femsched::Matrix>& ms) {
            std::vector<double> out;
            for (const auto& m : ms) out.insert(out.end(), m.data.begin(), m.data.end());
            return out;
        };
        for (std::size_t i = 0; i < sig.scalar_spaces.size(); ++i) phi_.push_back(flat(p.tabulations.scalar_phi.at(i)));
        for (std::size_t i = 0; i < sig.vector_spaces.size(); ++i) phi_.push_back(flat(p.tabulations.vector_phi.at(i)));
        psi_ = flat(p.tabulations.psi);
        std::size_t f = 0;
        for (std::size_t i = 0; i < sig.scalar_spaces.size(); ++i, ++f) {
            femgpu_space s{};
            s.dofs = sig.scalar_spaces[i].dofs;
            s.deriv_terms = sig.scalar_spaces[i].deriv_terms;
            s.phi = phi_[f].data();
            s.map = p.connectivity.scalar_maps.at(i).indices.data();
            s.global_count = p.connectivity.scalar_maps[i].global_count;
            s.input = p.scalar_inputs.at(i).data();
            scalar_.push_back(s);
        }
        for (std::size_t i = 0; i < sig.vector_spaces.size(); ++i, ++f) {
            femgpu_space s{};
            s.dofs = sig.vector_spaces[i].dofs;
            s.deriv_terms = sig.vector_spaces[i].deriv_terms;
            s.components = sig.vector_spaces[i].components.data();
            s.phi = phi_[f].data();
            s.map = p.connectivity.vector_maps.at(i).indices.data();
            s.global_count = p.connectivity.vector_maps[i].global_count;
            s.input = p.vector_inputs.at(i).data();
            vector_.push_back(s);
        }
        for (const auto& n : p.map.nodes()) {
            femgpu_map_node m{};
            m.op = static_cast<int32_t>(n.op);
            m.a = n.a;
            m.b = n.b;
            m.value = n.value;
            nodes_.push_back(m);
        }
        d_.dim = sig.dim;
        d_.quad_points = Q;
        d_.coord_dofs = sig.coord_dofs;
        d_.affine_geometry = sig.affine_geometry ? 1 : 0;
        d_.coordinate_space = sig.coordinate_space;
        d_.word_bytes = sig.word_bytes;
        d_.n_scalar = static_cast<int32_t>(scalar_.size());
        d_.n_vector = static_cast<int32_t>(vector_.size());
        d_.scalar_spaces = scalar_.data();
        d_.vector_spaces = vector_.data();
        d_.test_dofs = sig.test_dofs;
        d_.test_deriv_terms = sig.test_deriv_terms;
        d_.psi = psi_.data();
        d_.weights = p.tabulations.weights.data();
        d_.cell_count = p.connectivity.cell_count;
        d_.test_global_count = p.connectivity.test_map.global_count;
        d_.test_map = p.connectivity.test_map.indices.data();
        d_.coord_map = sig.affine_geometry ? p.connectivity.coord_map.indices.data() : nullptr;
        d_.coords = sig.affine_geometry ? p.connectivity.coords.data() : nullptr;
        d_.coord_global_count = p.connectivity.coord_global_count;
        d_.n_map_nodes = static_cast<int32_t>(nodes_.size());
        d_.map_nodes = nodes_.data();
        d_.map_outputs = p.map.outputs().data();
        d_.n_map_outputs = static_cast<int32_t>(p.map.outputs().size());
        d_.output_size = p.output_size;
    }
    const femgpu_problem* get() const { return &d_; }

private:
    std::vector<std::vector<double>> phi_;
    std::vector<double> psi_;
    std::vector<femgpu_space> scalar_, vector_;
    std::vector<femgpu_map_node> nodes_;
    femgpu_problem d_{};
};

// RAII device instance (femgpu_create/femgpu_destroy); re-blocking happens once here.
class DeviceInstance {
public:
    explicit DeviceInstance(const femsched::ProblemInstance& p) : output_size_(p.output_size) {
        ProblemView v(p);
        femgpu_instance* h = nullptr;
        check(femgpu_create(v.get(), &h));
        h_.reset(h);
    }
    std::vector<double> action(const femgpu_schedule* s = nullptr) {
        std::vector<double> y(static_cast<std::size_t>(output_size_));
        check(femgpu_action(h_.get(), s, y.data()));
        return y;
    }
    double measure(const femgpu_schedule* s = nullptr) {
        double sec = 0.0;
        check(femgpu_time_action(h_.get(), s, 5, 15, 0.2, &sec));
        return sec;
    }
    femgpu_instance* handle() const { return h_.get(); }

private:
    struct Del {
        void operator()(femgpu_instance* h) const { femgpu_destroy(h); }
    };
    std::unique_ptr<femgpu_instance, Del> h_;
    int output_size_;
};

// reference_action-shaped entry (form.hpp:471-472): same arguments, same return, same errors.
// counters, when given, are incremented exactly as reference_action increments them
// (femgpu_reference_counters: matvec mults/adds, map add/mul evaluations).
inline std::vector<double> action(const femsched::ProblemInstance& p, femsched::ReferenceCounters* counters = nullptr) {
    p.validate();  // identical argument checking to the reference, before any device work
    DeviceInstance d(p);
    std::vector<double> y = d.action();
    if (counters) {
        ProblemView v(p);
        int64_t m = 0, a = 0, o = 0;
        check(femgpu_reference_counters(v.get(), &m, &a, &o));
        counters->matvec_mults += m;
        counters->matvec_adds += a;
        counters->map_ops += o;
    }
    return y;
}

// Fused multi-operator action (femgpu_problem_fuse): instances on the same cells,
// geometry and quadrature run as one kernel; returns each instance's reference_action-shaped output.
inline std::vector<std::vector<double>> fused_action(const std::vector<const femsched::ProblemInstance*>& ps) {
    std::vector<std::unique_ptr<ProblemView>> views;
    std::vector<const femgpu_problem*> flat;
    for (const auto* p : ps) {
        p->validate();
        views.push_back(std::make_unique<ProblemView>(*p));
        flat.push_back(views.back()->get());
    }
    femgpu_owned_problem* own = nullptr;
    const femgpu_problem* fused = nullptr;
    std::vector<int64_t> off(ps.size() + 1);
    check(femgpu_problem_fuse(flat.data(), static_cast<int32_t>(flat.size()), &own, &fused, off.data()));
    std::unique_ptr<femgpu_owned_problem, femgpu_status (*)(femgpu_owned_problem*)> guard(own, femgpu_problem_free);
    femgpu_instance* h = nullptr;
    check(femgpu_create(fused, &h));
    std::unique_ptr<femgpu_instance, femgpu_status (*)(femgpu_instance*)> hg(h, femgpu_destroy);
    std::vector<double> y(static_cast<std::size_t>(off.back()));
    check(femgpu_action(h, nullptr, y.data()));
    std::vector<std::vector<double>> out;
    for (std::size_t i = 0; i < ps.size(); ++i) out.emplace_back(y.begin() + off[i], y.begin() + off[i + 1]);
    return out;
}

// Content fingerprint of an instance (sizes, maps, inputs, tabulations, map DAG): the executor's
// device-instance cache is keyed on it, not on the address, so an instance rebuilt at the same
// address or modified in place is re-uploaded.
inline uint64_t fingerprint(const femsched::ProblemInstance& p) {
    uint64_t h = 0xcbf29ce484222325ULL;
    auto mix = [&h](const void* data, std::size_t bytes) {
        const unsigned char* c = static_cast<const unsigned char*>(data);
        std::size_t i = 0;
        for (; i + 8 <= bytes; i += 8) {
            uint64_t w;
            std::memcpy(&w, c + i, 8);
            h = (h ^ w) * 0x100000001b3ULL;
            h ^= h >> 29;
        }
        for (; i < bytes; ++i) h = (h ^ c[i]) * 0x100000001b3ULL;
    };
    auto vec = [&](const auto& v) {
        const std::size_t n = v.size();
        mix(&n, sizeof n);
        if (n) mix(v.data(), n * sizeof(v[0]));
    };
    const auto& c = p.connectivity;
    mix(&c.cell_count, sizeof c.cell_count);
    mix(&p.output_size, sizeof p.output_size);
    for (const auto& m : c.scalar_maps) vec(m.indices);
    for (const auto& m : c.vector_maps) vec(m.indices);
    vec(c.test_map.indices);
    vec(c.coord_map.indices);
    vec(c.coords);
    for (const auto& x : p.scalar_inputs) vec(x);
    for (const auto& x : p.vector_inputs) vec(x);
    for (const auto& sp : p.tabulations.scalar_phi)
        for (const auto& m : sp) vec(m.data);
    for (const auto& sp : p.tabulations.vector_phi)
        for (const auto& m : sp) vec(m.data);
    for (const auto& m : p.tabulations.psi) vec(m.data);
    vec(p.tabulations.weights);
    for (const auto& n : p.map.nodes()) {
        const int v[3] = {static_cast<int>(n.op), n.a, n.b};
        mix(v, sizeof v);
        mix(&n.value, sizeof n.value);
    }
    vec(p.map.outputs());
    return h;
}

#ifdef FEMGPU_HAS_EXECUTOR
// TilingParams (qoi.hpp:23-33) -> femgpu_schedule.
inline femgpu_schedule schedule_from(const femsched::TilingParams& t) {
    femgpu_schedule s{};
    if (t.kind == femsched::ScheduleKind::SingleCellPerWorkItem) {
        s.kind = FEMGPU_SCPT;
        return s;
    }
    s.kind = FEMGPU_MLT;
    s.quad_tile = t.quad_tile;
    s.eval_row_tile = t.eval_row_tile;
    for (std::size_t i = 0; i < t.eval_col_tiles_scalar.size() && i < FEMGPU_MAX_SPACES; ++i)
        s.eval_col_tiles_scalar[i] = t.eval_col_tiles_scalar[i];
    for (std::size_t i = 0; i < t.eval_col_tiles_vector.size() && i < FEMGPU_MAX_SPACES; ++i)
        s.eval_col_tiles_vector[i] = t.eval_col_tiles_vector[i];
    s.quad_row_tile = t.quad_row_tile;
    s.quad_col_tile = t.quad_col_tile;
    s.cells_per_group = t.cells_per_group;
    s.lanes_per_cell = t.lanes_per_cell;
    return s;
}

// A measuring femsched::Executor (search.hpp:257-283) backed by the sm_100a kernels: uploads
// each instance once (tune calls it for b+1 candidates, possibly from std::async threads),
// verifies finiteness on the device, reports the CUDA-event mean of the paper's protocol.
inline femsched::Executor executor() {
    struct Cache {
        std::mutex mu;
        uint64_t key = 0;
        std::shared_ptr<DeviceInstance> dev;
    };
    auto cache = std::make_shared<Cache>();
    return [cache](const femsched::TilingParams& t, const femsched::ProblemInstance& inst) {
        femsched::ExecutionOutcome out;
        try {
            std::shared_ptr<DeviceInstance> d;
            {
                const uint64_t fp = fingerprint(inst);
                std::lock_guard<std::mutex> lk(cache->mu);
                if (cache->key != fp || !cache->dev) {
                    cache->dev = std::make_shared<DeviceInstance>(inst);
                    cache->key = fp;
                }
                d = cache->dev;
            }
            const femgpu_schedule s = schedule_from(t);
            out.output = d->action(&s);
            out.measured_seconds = d->measure(&s);
            // the execution census of the kernel that ran (femgpu_trace_counters)
            int64_t c[FEMGPU_TRACE_COUNTERS] = {};
            check(femgpu_trace_counters(d->handle(), &s, c, FEMGPU_TRACE_COUNTERS));
            out.counters.barriers_per_workgroup = c[0];
            out.counters.flops_matvec = c[1];
            out.counters.flops_masked_padding = c[2];
            out.counters.gather_words = c[3];
            out.counters.scatter_words = c[4];
            out.counters.reference_words = c[5];
            out.counters.reference_cached_words = c[6];
            out.counters.coord_words = c[7];
            out.counters.local_eval_read_words = c[8];
            out.counters.local_eval_write_words = c[9];
            out.counters.local_quad_read_words = c[10];
            out.counters.local_words_highwater = c[11];
            out.workgroups = c[12];
            out.ok = true;
        } catch (const std::exception& e) {
            out.error = e.what();  // search.hpp:278-280
        }
        return out;
    };
}
#endif

}  // namespace femgpu
