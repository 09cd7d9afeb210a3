// C++ drop-in test: femgpu::action vs femsched::reference_action (the reference's own code,
// compiled from /root/reference/proj/include), and femsched::tune with femgpu::executor().
// Built by tests/cpp/Makefile (needs the reference headers, so it is built in the container
// and the binary travels to the GPU box).  Exit code 0 = all checks passed; 77 = no GPU.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <unistd.h>

#define FEMGPU_WITH_FEMSCHED_SEARCH 1
#include <femgpu/femsched_adapter.hpp>

using namespace femsched;

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}

int main() {
    if (femgpu_device_count() < 1) {
        std::printf("no CUDA device: skipping\n");
        return 77;
    }
    int fails = 0;
    struct Case { Operator op; int d, p, q, cells; unsigned seed; };
    const Case cases[] = {{Operator::mass, 2, 2, 7, 16, 7}, {Operator::laplace, 2, 2, 6, 16, 7},
                          {Operator::helmholtz, 2, 3, 12, 16, 7}, {Operator::mass, 3, 1, 5, 16, 7},
                          {Operator::laplace, 3, 2, 8, 16, 7}, {Operator::helmholtz, 3, 1, 7, 16, 7},
                          {Operator::elasticity, 3, 2, 4, 60, 3}, {Operator::hyperelasticity, 2, 2, 6, 33, 5}};
    for (const auto& c : cases) {
        const auto sig = preset_signature(c.op, c.d, c.p, c.q);
        const auto inst = make_problem(sig, preset_map(c.op, sig), c.cells, c.seed);
        ReferenceCounters rc, gc;
        const auto ref = reference_action(inst, &rc);
        const auto got = femgpu::action(inst, &gc);
        const double err = rel_l2(got, ref);
        const bool cnt_ok = rc.matvec_mults == gc.matvec_mults && rc.matvec_adds == gc.matvec_adds && rc.map_ops == gc.map_ops;
        std::printf("%-16s d=%d p=%d Q=%2d cells=%3d  rel_l2=%.3e counters %s\n", operator_name(c.op), c.d, c.p, c.q,
                    c.cells, err, cnt_ok ? "equal" : "DIFFER");
        if (!(err <= 1e-12) || got.size() != ref.size() || !cnt_ok) ++fails;
    }
    // fused multi-operator action: stiffness and mass on one mesh, quadrature and trial vector
    {
        const auto sa = preset_signature(Operator::laplace, 3, 2, 8);
        const auto sb = preset_signature(Operator::mass, 3, 2, 8);
        const auto a = make_problem(sa, preset_map(Operator::laplace, sa), 40, 9);
        auto b = make_problem(sb, preset_map(Operator::mass, sb), 40, 9);
        b.tabulations.weights = a.tabulations.weights;
        b.connectivity.coords = a.connectivity.coords;
        b.connectivity.coord_map = a.connectivity.coord_map;
        b.connectivity.scalar_maps = a.connectivity.scalar_maps;
        b.connectivity.test_map = a.connectivity.test_map;
        b.scalar_inputs = a.scalar_inputs;
        b.output_size = a.output_size;
        const auto ys = femgpu::fused_action({&a, &b});
        const double ea = rel_l2(ys.at(0), reference_action(a)), eb = rel_l2(ys.at(1), reference_action(b));
        std::printf("fused laplace+mass: rel_l2 %.3e %.3e\n", ea, eb);
        if (!(ea <= 1e-12) || !(eb <= 1e-12)) ++fails;
    }
    // error mapping: invalid instance -> std::invalid_argument, NaN -> runtime_error naming the cell
    {
        const auto sig = preset_signature(Operator::mass, 2, 1, 2);
        auto inst = make_problem(sig, preset_map(Operator::mass, sig), 2, 1);
        inst.scalar_inputs[0][0] = std::nan("");
        std::string ref_msg, got_msg;
        try { reference_action(inst); } catch (const std::runtime_error& e) { ref_msg = e.what(); }
        try { femgpu::action(inst); } catch (const std::runtime_error& e) { got_msg = e.what(); }
        std::printf("non-finite: ref='%s' got='%s'\n", ref_msg.c_str(), got_msg.c_str());
        if (ref_msg != got_msg || ref_msg.empty()) ++fails;
    }
    // the executor's device-instance cache follows the instance's content, not its address: an
    // instance modified in place between calls is re-uploaded
    {
        const auto sig = preset_signature(Operator::laplace, 2, 2, 6);
        auto inst = make_problem(sig, preset_map(Operator::laplace, sig), 40, 9);
        auto ex = femgpu::executor();
        const auto a = ex(TilingParams::scpt(), inst);
        for (auto& v : inst.scalar_inputs[0]) v *= 2.0;
        const auto b = ex(TilingParams::scpt(), inst);
        const auto ref = reference_action(inst);
        const double err = a.ok && b.ok ? rel_l2(b.output, ref) : 1.0;
        std::printf("executor after in-place input change: rel_l2=%.3e\n", err);
        if (!(err <= 1e-12)) ++fails;
    }
    // tune through the measuring executor: b-best ranked MLT candidates + SCPT (search.hpp:338-416)
    {
        const auto sig = preset_signature(Operator::laplace, 2, 2, 6);
        const auto inst = make_problem(sig, preset_map(Operator::laplace, sig), 64, 7);
        SearchConfig cfg;
        cfg.best_count = 3;
        try {
            auto res = tune(inst, titan_v_device(), cfg, 1, femgpu::executor());
            std::printf("tune: %zu candidates verified, winner %s\n", res.records.size(),
                        detail::describe(res.winner.params).c_str());
            for (const auto& r : res.records)
                if (!r.output_ok || !std::isfinite(r.selection_seconds)) ++fails;
        } catch (const std::exception& e) {
            std::printf("tune failed: %s\n", e.what());
            ++fails;
        }
    }
    // the B200 DeviceSpec (devices/b200.device, measured on this GPU) feeding the
    // reference's own rank (b = 9 + SCPT) and tune through the measuring executor, jobs = 1 and 2
    // (search.hpp:396-403 calls the executor concurrently; results must not depend on jobs)
    {
        char exe[4096] = {0};
        const ssize_t n = readlink("/proc/self/exe", exe, sizeof exe - 1);
        std::string root = n > 0 ? std::string(exe, static_cast<size_t>(n)) : std::string();
        for (int up = 0; up < 4 && !root.empty(); ++up) root = root.substr(0, root.find_last_of('/'));
        std::ifstream is(root + "/devices/b200.device");
        if (!is) {
            std::printf("devices/b200.device missing\n");
            ++fails;
        } else {
            const DeviceSpec dev = load_device(is);
            const auto sig = preset_signature(Operator::elasticity, 3, 2, 4);
            const auto inst = make_problem(sig, preset_map(Operator::elasticity, sig), 200, 11);
            SearchConfig cfg;  // b = 9 (search.hpp defaults)
            try {
                auto r1 = tune(inst, dev, cfg, 1, femgpu::executor());
                auto r2 = tune(inst, dev, cfg, 2, femgpu::executor());
                std::printf("tune on %s: %zu candidates verified (jobs 1), %zu (jobs 2), winner %s\n", dev.name.c_str(),
                            r1.records.size(), r2.records.size(), detail::describe(r1.winner.params).c_str());
                if (r1.records.size() != r2.records.size()) ++fails;
                for (const auto* res : {&r1, &r2})
                    for (const auto& r : res->records)
                        if (!r.output_ok || !std::isfinite(r.selection_seconds)) ++fails;
            } catch (const std::exception& e) {
                std::printf("tune (b200) failed: %s\n", e.what());
                ++fails;
            }
        }
    }
    std::printf(fails ? "FAIL (%d)\n" : "PASS\n", fails);
    return fails ? 1 : 0;
}
