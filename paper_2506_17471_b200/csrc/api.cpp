// api.cpp — the extern "C" boundary (include/femgpu.h).  Converts every C++
// exception into a femgpu_status + thread-local message; nothing throws across.
#include <algorithm>
#include <cstring>
#include <fstream>
#include <string>

#include "femgpu_internal.hpp"


namespace {

thread_local std::string g_last_error;

}  // namespace

void femgpu::set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
thread_local int g_device = -1;

template <typename F>
femgpu_status guard(F&& f) {
    try {
        f();
        return FEMGPU_OK;
    } catch (const femgpu::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return FEMGPU_E_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FEMGPU_E_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return FEMGPU_E_INTERNAL;
    }
}

void bind_device() {
    if (g_device >= 0) FG_CUDA(cudaSetDevice(g_device));
}

femgpu::Instance& get(femgpu_instance* h) {
    if (!h || !h->impl) femgpu::invalid("null instance");
    return *h->impl;
}

void copy_inputs(femgpu::Instance& I, const double* const* scalar_inputs, const double* const* vector_inputs,
                 cudaStream_t stream) {
    for (size_t i = 0; i < I.sspaces.size(); ++i) {
        if (!scalar_inputs || !scalar_inputs[i]) femgpu::invalid("instance: scalar input length mismatch");
        FG_CUDA(cudaMemcpyAsync(I.sspaces[i].d_x, scalar_inputs[i], sizeof(double) * I.sspaces[i].global,
                                cudaMemcpyHostToDevice, stream));
    }
    for (size_t i = 0; i < I.vspaces.size(); ++i) {
        if (!vector_inputs || !vector_inputs[i]) femgpu::invalid("instance: vector input length mismatch");
        femgpu::upload_padded(I.vspaces[i].d_x, vector_inputs[i], I.vspaces[i].global, I.sig.dim, I.vspaces[i].d_stage,
                              stream);
    }
}

}  // namespace

extern "C" {

int32_t femgpu_abi_version(void) { return FEMGPU_ABI_VERSION; }

const char* femgpu_last_error(void) { return g_last_error.c_str(); }

int32_t femgpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

namespace {

// Buffer set b's device inputs swapped into the instance's spaces for the duration of a call
// (kernel parameters capture the pointers at launch).
void swap_inputs(femgpu::Instance& I, int b) {
    if (b != 1) return;
    const size_t n = I.sspaces.size() + I.vspaces.size();
    if (I.x_alt.empty()) {
        const int vs = femgpu::vec_stride(I.sig.dim);
        for (const auto& sp : I.sspaces) I.x_alt.push_back(I.alloc<double>(static_cast<size_t>(sp.global)));
        for (const auto& sp : I.vspaces) I.x_alt.push_back(I.alloc<double>(static_cast<size_t>(sp.global) * vs));
    }
    for (size_t i = 0; i < n; ++i) {
        auto& ds = i < I.sspaces.size() ? I.sspaces[i] : I.vspaces[i - I.sspaces.size()];
        std::swap(ds.d_x, I.x_alt[i]);
    }
}

// Completes the streaming steps: both sets' downloads and computes; the instance then holds the last
// step's inputs and output (set 1 copied into set 0), and a non-finite value in any step is reported
// (diagnosed on the last step's inputs).
void async_drain(femgpu::Instance& I) {
    if (I.async_pending == 0) return;
    FG_CUDA(cudaStreamSynchronize(I.s_d2h));
    FG_CUDA(cudaStreamSynchronize(I.stream));
    if (I.async_last == 1) {
        const int vs = femgpu::vec_stride(I.sig.dim);
        size_t i = 0;
        for (auto& sp : I.sspaces)
            FG_CUDA(cudaMemcpyAsync(sp.d_x, I.x_alt[i++], sizeof(double) * sp.global, cudaMemcpyDeviceToDevice, I.stream));
        for (auto& sp : I.vspaces)
            FG_CUDA(cudaMemcpyAsync(sp.d_x, I.x_alt[i++], sizeof(double) * sp.global * vs, cudaMemcpyDeviceToDevice, I.stream));
        FG_CUDA(cudaMemcpyAsync(I.d_y, I.second_output(), sizeof(double) * static_cast<size_t>(I.output_size),
                                cudaMemcpyDeviceToDevice, I.stream));
    }
    I.async_pending = 0;
    I.async_used[0] = I.async_used[1] = false;
    I.async_next = 0;
    femgpu::check_failure(I, I.async_kp, I.stream);
}

}  // namespace

femgpu_status femgpu_set_device(int32_t device) {
    return guard([&] {
        FG_CUDA(cudaSetDevice(device));
        g_device = device;
    });
}

femgpu_status femgpu_usable_flops(const femgpu_problem* p, int64_t* flops) {
    return guard([&] {
        if (!p || !flops) femgpu::invalid("null argument");
        femgpu::validate_problem(p);
        *flops = femgpu::signature_from(p).usable_flops();
    });
}

femgpu_status femgpu_reference_counters(const femgpu_problem* p, int64_t* matvec_mults, int64_t* matvec_adds,
                                        int64_t* map_ops) {
    return guard([&] {
        if (!p) femgpu::invalid("null argument");
        femgpu::validate_problem(p);
        // reference_action's ReferenceCounters (form.hpp:463-472, counted at :534-537, :550-553,
        // :571, :582-585): per cell and quadrature point one mult + one add per Phi entry of every
        // trial term and per (test dof, test term); map_ops counts the add/mul nodes the unmemoised
        // recursive eval_node (form.hpp:298-318) visits, i.e. the expression-tree size of each output
        std::vector<long long> tree(static_cast<size_t>(p->n_map_nodes), 0);
        for (int id = 0; id < p->n_map_nodes; ++id) {
            const femgpu_map_node& n = p->map_nodes[id];
            if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) tree[id] = 1 + tree[n.a] + tree[n.b];
        }
        long long per_qp = 0, map = 0;
        for (int i = 0; i < p->n_scalar; ++i) per_qp += static_cast<long long>(p->scalar_spaces[i].deriv_terms) * p->scalar_spaces[i].dofs;
        for (int i = 0; i < p->n_vector; ++i) per_qp += static_cast<long long>(p->vector_spaces[i].deriv_terms) * p->vector_spaces[i].dofs;
        per_qp += static_cast<long long>(p->test_dofs) * p->test_deriv_terms;
        for (int k = 0; k < p->n_map_outputs; ++k) map += tree[p->map_outputs[k]];
        const long long cq = static_cast<long long>(p->cell_count) * p->quad_points;
        if (matvec_mults) *matvec_mults = cq * per_qp;
        if (matvec_adds) *matvec_adds = cq * per_qp;
        if (map_ops) *map_ops = cq * map;
    });
}

femgpu_status femgpu_validate(const femgpu_problem* p) {
    return guard([&] { femgpu::validate_problem(p); });
}

femgpu_status femgpu_emit_source(const femgpu_problem* p, const femgpu_schedule* s, char* buf, size_t cap,
                                 size_t* len) {
    return guard([&] {
        femgpu::validate_problem(p);
        femgpu::Signature sig = femgpu::signature_from(p);
        // Host-only resolution (no device instance): SCPT with global atomics, or MLT.
        femgpu::KernelPlan kp;
        if (s && s->kind == FEMGPU_DMMA) {
            femgpu::resolve_dmma(sig, kp, s);
            // emitter checks without an instance: assume an interleaved vector test space when
            // the shapes allow it (the instance decides from the actual maps)
            for (int i = 0; i < sig.nv() && kp.tvec < 0; ++i)
                if (sig.vdofs[i] * sig.dim == sig.nW) kp.tvec = i;
        } else if (s && s->kind == FEMGPU_MLT) {
            kp.family = femgpu::Family::Mlt;
            kp.TQ = s->quad_tile;
            kp.Ter = s->eval_row_tile;
            kp.Tqr = s->quad_row_tile;
            kp.Tqc = s->quad_col_tile;
            kp.Nc = s->cells_per_group;
            kp.Nwi = s->lanes_per_cell;
            kp.block = kp.Nc * kp.Nwi;
            kp.basis = FEMGPU_BASIS_SMEM;
            for (int i = 0; i < sig.ns(); ++i) kp.Tcs.push_back(s->eval_col_tiles_scalar[i]);
            for (int i = 0; i < sig.nv(); ++i) kp.Tcv.push_back(s->eval_col_tiles_vector[i]);
        } else {
            kp.family = femgpu::Family::Scpt;
            kp.basis = (s && s->basis) ? s->basis : (sig.tab_size <= 512 ? FEMGPU_BASIS_CONST : FEMGPU_BASIS_SMEM);
            kp.block = (s && s->block_cells > 0) ? s->block_cells : 128;
            if (s && s->scatter == FEMGPU_SCATTER_TILE) femgpu::host_tile_plan(p, sig, kp, s);
            if (s && s->scatter == FEMGPU_SCATTER_MACRO) femgpu::host_macro_plan(p, sig, kp, s);
            if (s && s->scatter == FEMGPU_SCATTER_ATOMIC && s->group_cells > 1) kp.G = s->group_cells;
            if (s && (s->reserved[3] & 0xff) == 4) kp.qloop = true;
            if (s && s->scatter == FEMGPU_SCATTER_COLOR) kp.colour = true;
        }
        kp.strict = s && (s->reserved[0] & FEMGPU_FLAG_STRICT);
        femgpu::EmitResult em = femgpu::emit_kernel(sig, kp);
        if (len) *len = em.source.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, em.source.size());
            std::memcpy(buf, em.source.data(), n);
            buf[n] = 0;
        }
    });
}

femgpu_status femgpu_jit_check(const femgpu_problem* p, const femgpu_schedule* s) {
    return guard([&] {
        size_t len = 0;
        femgpu_status st = femgpu_emit_source(p, s, nullptr, 0, &len);
        if (st != FEMGPU_OK) throw femgpu::Error(st, g_last_error);
        std::string src(len + 1, '\0');
        femgpu_emit_source(p, s, src.data(), src.size(), &len);
        src.resize(len);
        std::string log;
        femgpu::jit_compile(src, s && (s->reserved[0] & FEMGPU_FLAG_STRICT), &log);
    });
}

femgpu_status femgpu_create(const femgpu_problem* p, femgpu_instance** out) {
    return guard([&] {
        if (!out) femgpu::invalid("null output handle");
        *out = nullptr;
        bind_device();
        auto h = new femgpu_instance;
        try {
            h->impl = femgpu::create_instance(p);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

femgpu_status femgpu_destroy(femgpu_instance* inst) {
    return guard([&] { delete inst; });
}

femgpu_status femgpu_set_inputs(femgpu_instance* h, const double* const* scalar_inputs,
                                const double* const* vector_inputs) {
    return guard([&] {
        auto& I = get(h);
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        copy_inputs(I, scalar_inputs, vector_inputs, I.stream);
        FG_CUDA(cudaStreamSynchronize(I.stream));
    });
}

femgpu_status femgpu_action(femgpu_instance* h, const femgpu_schedule* s, double* y_host) {
    return guard([&] {
        auto& I = get(h);
        if (!y_host) femgpu::invalid("null output buffer");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        femgpu::run_action(I, kp, I.d_y, I.stream);
        FG_CUDA(cudaMemcpyAsync(y_host, I.d_y, sizeof(double) * static_cast<size_t>(I.output_size),
                                cudaMemcpyDeviceToHost, I.stream));
        femgpu::check_failure(I, kp, I.stream);
    });
}

femgpu_status femgpu_action_host(femgpu_instance* h, const femgpu_schedule* s, const double* const* scalar_inputs,
                                 const double* const* vector_inputs, double* y_host) {
    return guard([&] {
        auto& I = get(h);
        if (!y_host) femgpu::invalid("null output buffer");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        // overlapped H2D / slabs / D2H when the instance has locality (pipeline.cpp), else sequential
        if (!femgpu::pipelined_host_action(I, kp, scalar_inputs, vector_inputs, y_host)) {
            copy_inputs(I, scalar_inputs, vector_inputs, I.stream);
            femgpu::run_action(I, kp, I.d_y, I.stream);
            FG_CUDA(cudaMemcpyAsync(y_host, I.d_y, sizeof(double) * static_cast<size_t>(I.output_size),
                                    cudaMemcpyDeviceToHost, I.stream));
        }
        femgpu::check_failure(I, kp, I.stream);
    });
}

femgpu_status femgpu_action_host_async(femgpu_instance* h, const femgpu_schedule* s, const double* const* scalar_inputs,
                                       const double* const* vector_inputs, double* y_host) {
    return guard([&] {
        auto& I = get(h);
        if (!y_host) femgpu::invalid("null output buffer");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        if (!s && !I.auto_ready) async_drain(I);  // the automatic schedule's timing pass uses the instance buffers
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        if (I.async_pending && kp.key() != I.async_kp.key()) async_drain(I);  // one schedule per stream of steps
        const int b = I.async_next;
        swap_inputs(I, b);
        bool ok = false;
        try {
            ok = femgpu::pipelined_host_action(I, kp, scalar_inputs, vector_inputs, y_host, b,
                                               b ? I.second_output() : I.d_y);
        } catch (...) {
            swap_inputs(I, b);
            throw;
        }
        swap_inputs(I, b);
        if (!ok) {  // no slab plan for this instance: a synchronous step
            async_drain(I);
            copy_inputs(I, scalar_inputs, vector_inputs, I.stream);
            femgpu::run_action(I, kp, I.d_y, I.stream);
            FG_CUDA(cudaMemcpyAsync(y_host, I.d_y, sizeof(double) * static_cast<size_t>(I.output_size),
                                    cudaMemcpyDeviceToHost, I.stream));
            femgpu::check_failure(I, kp, I.stream);
            return;
        }
        I.async_kp = kp;
        I.async_last = b;
        I.async_next = b ^ 1;
        ++I.async_pending;
    });
}

femgpu_status femgpu_action_host_wait(femgpu_instance* h) {
    return guard([&] {
        auto& I = get(h);
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);
    });
}

femgpu_status femgpu_cg(femgpu_instance* h, const femgpu_schedule* s, const double* b_dev, double* x_dev, double rtol,
                        int32_t maxiter, int32_t check_every, int32_t* iterations, double* rel_residual) {
    return guard([&] {
        auto& I = get(h);
        if (!b_dev || !x_dev) femgpu::invalid("cg: null vector");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        int it = 0;
        femgpu::device_cg(I, kp, b_dev, x_dev, rtol, maxiter, check_every, &it, rel_residual);
        if (iterations) *iterations = it;
    });
}

femgpu_status femgpu_action_device(femgpu_instance* h, const femgpu_schedule* s, double* y_dev, void* stream) {
    return guard([&] {
        auto& I = get(h);
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        femgpu::run_action(I, kp, y_dev ? y_dev : I.d_y, stream ? static_cast<cudaStream_t>(stream) : I.stream);
    });
}

femgpu_status femgpu_action_device_pipelined(femgpu_instance* h, const femgpu_schedule* s, double* y_dev,
                                             double* y_next_dev, void* stream) {
    return guard([&] {
        auto& I = get(h);
        if (!y_dev) femgpu::invalid("action_device_pipelined: null output buffer");
        if (y_next_dev == y_dev) femgpu::invalid("action_device_pipelined: y_next must not alias y");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        femgpu::run_action_pipelined(I, kp, y_dev, y_next_dev, stream ? static_cast<cudaStream_t>(stream) : I.stream);
    });
}

femgpu_status femgpu_check_finite(femgpu_instance* h, const femgpu_schedule* s, void* stream) {
    return guard([&] {
        auto& I = get(h);
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        femgpu::check_failure(I, kp, stream ? static_cast<cudaStream_t>(stream) : I.stream);
    });
}

femgpu_status femgpu_time_action(femgpu_instance* h, const femgpu_schedule* s, int32_t warmup, int32_t min_reps,
                                 double min_seconds, double* seconds) {
    return guard([&] {
        auto& I = get(h);
        if (!seconds) femgpu::invalid("null output");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        for (int i = 0; i < warmup; ++i) femgpu::run_action(I, kp, I.d_y, I.stream);
        femgpu::check_failure(I, kp, I.stream);
        double total = 0.0;
        long long reps = 0;
        int batch = std::max(1, min_reps);
        while (reps < min_reps || total < min_seconds) {
            FG_CUDA(cudaEventRecord(I.ev0, I.stream));
            for (int i = 0; i < batch; ++i) femgpu::run_action(I, kp, I.d_y, I.stream);
            FG_CUDA(cudaEventRecord(I.ev1, I.stream));
            FG_CUDA(cudaEventSynchronize(I.ev1));
            float ms = 0.f;
            FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
            total += ms * 1e-3;
            reps += batch;
            if (reps > 1000000) break;
        }
        femgpu::check_failure(I, kp, I.stream);
        *seconds = total / static_cast<double>(reps);
    });
}

femgpu_status femgpu_time_steps(femgpu_instance* h, const femgpu_schedule* s, int32_t steps, double* seconds) {
    return femgpu_time_steps_ex(h, s, steps, 0, seconds);
}

femgpu_status femgpu_time_steps_ex(femgpu_instance* h, const femgpu_schedule* s, int32_t steps, int32_t flags,
                                   double* seconds) {
    return guard([&] {
        auto& I = get(h);
        if (steps < 1 || !seconds) femgpu::invalid("time_steps: steps >= 1 and an output are required");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        const bool piped = (flags & FEMGPU_STEPS_PIPELINED) != 0;
        double* ybuf[2] = {I.d_y, piped ? I.second_output() : I.d_y};
        if (piped) {  // the first step's output is zeroed outside the timed region, as the previous step would
            FG_CUDA(cudaMemsetAsync(ybuf[0], 0, sizeof(double) * static_cast<size_t>(I.output_size), I.stream));
            femgpu::run_action_pipelined(I, kp, ybuf[0], ybuf[1], I.stream);  // warm (JIT of the zeroing variant)
            FG_CUDA(cudaMemsetAsync(ybuf[0], 0, sizeof(double) * static_cast<size_t>(I.output_size), I.stream));
        }
        FG_CUDA(cudaDeviceSynchronize());
        FG_CUDA(cudaEventRecord(I.ev0, I.stream));
        for (int i = 0; i < steps; ++i) {
            if (piped)
                femgpu::run_action_pipelined(I, kp, ybuf[i & 1], ybuf[(i + 1) & 1], I.stream);
            else
                femgpu::run_action(I, kp, I.d_y, I.stream);
        }
        FG_CUDA(cudaEventRecord(I.ev1, I.stream));
        FG_CUDA(cudaEventSynchronize(I.ev1));
        FG_CUDA(cudaDeviceSynchronize());
        float ms = 0.f;
        FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
        if (piped && ((steps - 1) & 1))  // the last step wrote the second buffer: device_output shows it
            FG_CUDA(cudaMemcpyAsync(I.d_y, ybuf[1], sizeof(double) * static_cast<size_t>(I.output_size),
                                    cudaMemcpyDeviceToDevice, I.stream));
        femgpu::check_failure(I, kp, I.stream);
        *seconds = ms * 1e-3;
    });
}

femgpu_status femgpu_profile_action(femgpu_instance* h, const femgpu_schedule* s, int32_t warmup, int32_t reps,
                                    double* step_seconds, double* kernel_seconds, double* zero_seconds) {
    return guard([&] {
        auto& I = get(h);
        if (reps < 1) femgpu::invalid("profile: reps must be >= 1");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        for (int i = 0; i < warmup; ++i) femgpu::run_action(I, kp, I.d_y, I.stream);
        femgpu::check_failure(I, kp, I.stream);
        std::vector<cudaEvent_t> ev(3 * static_cast<size_t>(reps));
        for (auto& e : ev) FG_CUDA(cudaEventCreate(&e));
        for (int i = 0; i < reps; ++i) {
            FG_CUDA(cudaEventRecord(ev[3 * i], I.stream));
            femgpu::run_action(I, kp, I.d_y, I.stream, ev[3 * i + 1]);
            FG_CUDA(cudaEventRecord(ev[3 * i + 2], I.stream));
        }
        FG_CUDA(cudaEventSynchronize(ev.back()));
        double step = 0, kern = 0, zero = 0;
        for (int i = 0; i < reps; ++i) {
            float a = 0, b = 0, c = 0;
            FG_CUDA(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 2]));
            FG_CUDA(cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]));
            FG_CUDA(cudaEventElapsedTime(&c, ev[3 * i], ev[3 * i + 1]));
            step += a;
            kern += b;
            zero += c;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        femgpu::check_failure(I, kp, I.stream);
        if (step_seconds) *step_seconds = step * 1e-3 / reps;
        if (kernel_seconds) *kernel_seconds = kern * 1e-3 / reps;
        if (zero_seconds) *zero_seconds = zero * 1e-3 / reps;
    });
}

femgpu_status femgpu_execute(femgpu_instance* h, const femgpu_schedule* s, double* y_host, double* measured) {
    femgpu_status st = femgpu_action(h, s, y_host);
    if (st != FEMGPU_OK) return st;
    if (measured) return femgpu_time_action(h, s, 5, 15, 0.2, measured);
    return FEMGPU_OK;
}

femgpu_status femgpu_default_schedule(const femgpu_instance* h, femgpu_schedule* s) {
    return guard([&] {
        if (!h || !h->impl || !s) femgpu::invalid("null argument");
        auto& I = *h->impl;  // the automatic schedule is a lazily computed cache of the instance
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        if (!I.auto_ready) {
            async_drain(I);  // the timing pass uses the instance buffers
            femgpu::autotune(I);
        }
        *s = I.auto_sched;
    });
}

femgpu_status femgpu_describe_schedule(femgpu_instance* h, const femgpu_schedule* s, char* buf, size_t cap,
                                       size_t* len) {
    return guard([&] {
        auto& I = get(h);
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        if (!s && !I.auto_ready) async_drain(I);
        std::string d = femgpu::describe_plan(femgpu::plan_for(I, s));
        if (!s) d += " | auto: " + I.auto_log;
        if (len) *len = d.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, d.size());
            std::memcpy(buf, d.data(), n);
            buf[n] = 0;
        }
    });
}

femgpu_status femgpu_stats(const femgpu_instance* h, int64_t* launches, int64_t* device_bytes, int64_t* tiles,
                           int64_t* max_tile_dofs) {
    return guard([&] {
        if (!h || !h->impl) femgpu::invalid("null instance");
        const auto& I = *h->impl;
        if (launches) *launches = I.last_launches;
        if (device_bytes) *device_bytes = I.device_bytes;
        int64_t nt = 0, mx = 0;
        for (const auto& kv : I.tiles) {
            nt = kv.second->n_tiles;
            mx = kv.second->groups.empty() ? 0 : kv.second->groups[I.test_group].max_unique;
        }
        if (tiles) *tiles = nt;
        if (max_tile_dofs) *max_tile_dofs = mx;
    });
}

femgpu_status femgpu_trace_counters(femgpu_instance* h, const femgpu_schedule* s, int64_t* out, int32_t n) {
    return guard([&] {
        auto& I = get(h);
        if (!out || n < FEMGPU_TRACE_COUNTERS) femgpu::invalid("trace_counters: need FEMGPU_TRACE_COUNTERS outputs");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        const femgpu::KernelPlan kp = femgpu::plan_for(I, s);
        auto mod = I.module_for(kp);
        const femgpu::Signature& sig = I.sig;
        const long long C = I.cells, d = sig.dim;
        int64_t c[FEMGPU_TRACE_COUNTERS] = {};
        const bool staged = kp.basis == FEMGPU_BASIS_SMEM || kp.family == femgpu::Family::Dmma ||
                            kp.family == femgpu::Family::Mlt;
        c[0] = staged ? 1 : 0;                                              // barriers per workgroup
        c[1] = sig.usable_flops() * C;                                      // flops_matvec
        if (kp.family == femgpu::Family::Dmma) {                            // flops_masked_padding
            const femgpu::DmmaLayout L = femgpu::dmma_layout(sig, kp);
            c[2] = std::max<long long>(0, L.nfrag * 64 - sig.usable_flops()) * C;
        }
        long long gather = 0, coord = 0, scatter = 0;
        if (kp.family == femgpu::Family::Macro) {  // unique nodes of each group, once
            const femgpu::MacroLayout& M = I.macro_layout(kp.G);
            const long long ng = C / kp.G;
            for (size_t i = 0; i < I.sspaces.size(); ++i) gather += M.unique[I.sspaces[i].group] * ng;
            for (size_t i = 0; i < I.vspaces.size(); ++i) gather += d * M.unique[I.vspaces[i].group] * ng;
            if (sig.affine) coord = d * M.unique[I.coord_group] * ng;
            scatter = static_cast<long long>(M.unique[I.test_group]) * ng;
        } else {
            for (int i = 0; i < sig.ns(); ++i) gather += static_cast<long long>(sig.sdofs[i]) * C;
            for (int i = 0; i < sig.nv(); ++i) gather += d * sig.vdofs[i] * C;
            if (sig.affine) coord = static_cast<long long>(sig.coord_dofs) * d * C;
            scatter = static_cast<long long>(sig.nW) * C;
        }
        const long long grid = femgpu::launch_grid(I, kp, *mod, C);
        c[3] = gather;                                                      // gather_words
        c[4] = scatter;                                                     // scatter_words (red.add)
        c[5] = kp.basis == FEMGPU_BASIS_CONST ? 0 : sig.tab_size * grid;    // reference_words (staged per CTA)
        c[6] = kp.basis == FEMGPU_BASIS_CONST ? sig.tab_size * C : 0;       // reference_cached_words (constant bank)
        c[7] = coord;                                                       // coord_words
        c[11] = static_cast<long long>(mod->emitted.smem_bytes / 8);        // local_words_highwater
        c[12] = grid;                                                       // workgroups (CTAs)
        std::copy(c, c + FEMGPU_TRACE_COUNTERS, out);
    });
}

femgpu_status femgpu_read_output(femgpu_instance* h, double* y_host) {
    return guard([&] {
        auto& I = get(h);
        if (!y_host) femgpu::invalid("null output buffer");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first
        FG_CUDA(cudaMemcpyAsync(y_host, I.d_y, sizeof(double) * static_cast<size_t>(I.output_size),
                                cudaMemcpyDeviceToHost, I.stream));
        FG_CUDA(cudaStreamSynchronize(I.stream));
    });
}

femgpu_status femgpu_device_output(femgpu_instance* h, double** y_dev) {
    return guard([&] {
        auto& I = get(h);
        if (!y_dev) femgpu::invalid("device_output: null output pointer");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first: d_y then holds the last step's output
        *y_dev = I.d_y;
    });
}

femgpu_status femgpu_device_input(femgpu_instance* h, int32_t space, double** x_dev) {
    return guard([&] {
        auto& I = get(h);
        const int ns = static_cast<int>(I.sspaces.size()), nv = static_cast<int>(I.vspaces.size());
        if (!x_dev || space < 0 || space >= ns + nv) femgpu::invalid("device_input: space out of range");
        std::lock_guard<std::mutex> lk(I.mu);
        FG_CUDA(cudaSetDevice(I.device));
        async_drain(I);  // streaming steps complete first: the caller may write the buffer next
        *x_dev = space < ns ? I.sspaces[space].d_x : I.vspaces[space - ns].d_x;
    });
}

femgpu_status femgpu_stream(femgpu_instance* h, void** stream) {
    return guard([&] { *stream = get(h).stream; });
}

femgpu_status femgpu_action_once(const femgpu_problem* p, double* y_host) {
    femgpu_instance* h = nullptr;
    femgpu_status st = femgpu_create(p, &h);
    if (st != FEMGPU_OK) return st;
    st = femgpu_action(h, nullptr, y_host);
    std::string err = g_last_error;
    femgpu_destroy(h);
    g_last_error = err;
    return st;
}

femgpu_status femgpu_problem_load(const char* path, femgpu_owned_problem** out, const femgpu_problem** view) {
    return guard([&] {
        if (!path || !out || !view) femgpu::invalid("null argument");
        std::ifstream is(path, std::ios::binary);
        if (!is) femgpu::invalid(std::string("cannot open: ") + path);
        femgpu_owned_problem* p = femgpu::load_problem(is);
        *out = p;
        *view = femgpu_owned_view(p);
    });
}

femgpu_status femgpu_problem_free(femgpu_owned_problem* p) {
    return guard([&] { femgpu_owned_delete(p); });
}

femgpu_status femgpu_problem_save(const femgpu_problem* p, const char* path) {
    return guard([&] {
        if (!p || !path) femgpu::invalid("null argument");
        std::ofstream os(path, std::ios::binary);
        if (!os) femgpu::invalid(std::string("cannot open for writing: ") + path);
        femgpu::save_problem(os, p);
        if (!os) femgpu::invalid(std::string("write failed: ") + path);
    });
}

femgpu_status femgpu_schedule_save(const femgpu_schedule* s, int32_t n_scalar, int32_t n_vector, const char* path) {
    return guard([&] {
        if (!s || !path) femgpu::invalid("null argument");
        if (n_scalar < 0 || n_vector < 0 || n_scalar > FEMGPU_MAX_SPACES || n_vector > FEMGPU_MAX_SPACES)
            femgpu::invalid("candidate file: bad space counts");
        std::ofstream os(path, std::ios::binary);
        if (!os) femgpu::invalid(std::string("cannot open for writing: ") + path);
        femgpu::save_schedule(os, s, n_scalar, n_vector);
    });
}

femgpu_status femgpu_schedule_load(const char* path, femgpu_schedule* s) {
    return guard([&] {
        if (!path || !s) femgpu::invalid("null argument");
        std::ifstream is(path, std::ios::binary);
        if (!is) femgpu::invalid(std::string("cannot open: ") + path);
        *s = femgpu::load_schedule(is);
    });
}

femgpu_status femgpu_host_alloc(size_t bytes, void** ptr) {
    return guard([&] { FG_CUDA(cudaMallocHost(ptr, bytes)); });
}

femgpu_status femgpu_host_free(void* ptr) {
    return guard([&] { FG_CUDA(cudaFreeHost(ptr)); });
}

}  // extern "C"
