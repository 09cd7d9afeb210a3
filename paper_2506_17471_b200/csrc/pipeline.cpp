// pipeline.cpp — end-to-end action with host buffers (femgpu_action_host) overlapped across
// three streams: the inputs are uploaded in node-ordered chunks, the action runs slab by slab
// over contiguous cell ranges as soon as the nodes a slab reads are resident, and the finished
// part of y is downloaded while later slabs still compute.  PCIe is full duplex, so the H2D of x
// and the D2H of y overlap each other and the kernels: the host-buffer action approaches
// max(H2D, D2H) instead of H2D + action + D2H.
//
// The slab plan comes from the instance's own maps (no mesh assumptions): for slab k and every
// distinct map, the min/max index its cells touch.  Inputs of space i must be resident up to
// max_k (prefix maximum); y rows below the smallest index any later slab touches are final after
// slab k (suffix minimum) and are downloaded then; y rows are zeroed just before the first slab
// that can write them.  Brick-major structured meshes give near-ideal overlap; for an instance
// without locality the plan degenerates to the sequential order (and is then not used).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <limits>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

constexpr long long kPipeMinCells = 1000000;
constexpr long long kZeroOverlapMinRows = 1 << 21;  // 16 MB of y: ~3 us of memset
constexpr long long kZeroOverlapMinCells = 1 << 16;

// Slabs of the overlapped host-buffer action: FEMGPU_PIPE_SLABS, else ~1 per 0.9 M cells in [4, 16].
// Each slab costs ~11 us (a sub-wave kernel tail plus its copies and events): C2 (7.35 M cells)
// e2e 2.265 / 2.227 / 2.302 / 2.601 / 2.828 ms at 4 / 8 / 16 / 32 / 64 slabs (tools/e2e_slabs.py).
int slab_count(long long cells) {
    const char* e = std::getenv("FEMGPU_PIPE_SLABS");
    const long long k = e ? std::atoi(e) : std::max(4LL, std::min(16LL, (cells + 450000) / 900000));
    return static_cast<int>(std::max(2LL, std::min(128LL, k)));
}

// slabs for fused zeroing: FEMGPU_ZERO_SLABS, else the schedule's count (reserved[0] >> 8), else 8
int zero_slab_count(int sched_slabs) {
    const char* e = std::getenv("FEMGPU_ZERO_SLABS");
    const int k = e ? std::atoi(e) : (sched_slabs > 0 ? sched_slabs : 8);
    return std::max(2, std::min(64, k));
}

}  // namespace

const PipePlan& Instance::pipe_plan(int align) {
    const int K = slab_count(cells);
    if (pipe && pipe->align == align && static_cast<int>(pipe->cb.size()) == K + 1) return *pipe;
    pipe = slab_plan(K, align);
    return *pipe;
}

// Streaming steps (femgpu_action_host_async) overlap one step's download with the next step's upload,
// so fill and drain are hidden and per-slab costs dominate: 2 slabs by default
// (C2: 1.775 / 1.884 / 2.016 ms per step at 2 / 4 / 8 slabs; FEMGPU_STREAM_SLABS overrides).
const PipePlan& Instance::stream_plan(int align) {
    const char* e = std::getenv("FEMGPU_STREAM_SLABS");
    const int K = std::max(2, std::min(128, e ? std::atoi(e) : 2));
    if (pipe_stream && pipe_stream->align == align && static_cast<int>(pipe_stream->cb.size()) == K + 1) return *pipe_stream;
    pipe_stream = slab_plan(K, align);
    return *pipe_stream;
}

const PipePlan& Instance::zero_plan(int align, int slabs, int max_slabs) {
    const int K = std::min(zero_slab_count(slabs), std::max(2, max_slabs));
    auto& z = zplans[{align, K}];
    if (!z) z = slab_plan(K, align);
    return *z;
}

std::unique_ptr<PipePlan> Instance::slab_plan(int K, int align) const {
    auto P = std::make_unique<PipePlan>();
    P->align = align;
    // slab sizes: equal by default; FEMGPU_PIPE_EDGE scales the first and last (fill / drain)
    const long long units = (static_cast<long long>(cells) + align - 1) / align;
    const char* edge_env = std::getenv("FEMGPU_PIPE_EDGE");
    const double edge = edge_env ? std::atof(edge_env) : 1.0;  // measured: half-size edges do not help (PCIe-bound)
    const double total_w = (K - 2) + 2 * edge;
    double acc = 0.0;
    P->cb.push_back(0);
    for (int k = 0; k < K; ++k) {
        acc += (k == 0 || k == K - 1) ? edge : 1.0;
        const long long u = k == K - 1 ? units : static_cast<long long>(units * acc / total_w);
        P->cb.push_back(static_cast<int>(std::min<long long>(cells, u * align)));
    }
    const size_t ng = group_maps.size();
    std::vector<std::vector<long long>> lo(ng, std::vector<long long>(K)), hi(ng, std::vector<long long>(K));
    for (size_t g = 0; g < ng; ++g) {
        const std::vector<int32_t>& m = group_maps[g];
        const long long E = static_cast<long long>(m.size() / cells);
        for (int k = 0; k < K; ++k) {
            long long a = std::numeric_limits<long long>::max(), b = -1;
            for (long long i = static_cast<long long>(P->cb[k]) * E; i < static_cast<long long>(P->cb[k + 1]) * E; ++i) {
                a = std::min<long long>(a, m[i]);
                b = std::max<long long>(b, m[i]);
            }
            lo[g][k] = b < 0 ? group_global[g] : a;
            hi[g][k] = b + 1;
        }
    }
    auto prefix_max = [&](int g) {
        std::vector<long long> v(K);
        long long run = 0;
        for (int k = 0; k < K; ++k) v[k] = run = std::max(run, hi[g][k]);
        return v;
    };
    for (const auto& sp : sspaces) P->up.push_back(prefix_max(sp.group));
    for (const auto& sp : vspaces) P->up.push_back(prefix_max(sp.group));
    P->zero_hi = prefix_max(test_group);
    P->zero_hi[K - 1] = output_size;  // rows no cell touches are zeros of the result too
    P->fin.assign(K, output_size);
    long long run = output_size;
    for (int k = K - 1; k >= 0; --k) {
        P->fin[k] = run;
        run = std::min(run, lo[test_group][k]);
    }
    // rows no cell touches (a gap in the test numbering) are final early but only zeroed when the
    // zeroing front reaches them: never download a row before it is zeroed
    for (int k = 0; k < K; ++k) P->fin[k] = std::min(P->fin[k], P->zero_hi[k]);
    // useful when the first slab needs a small part of the inputs and y completes progressively
    long long need0 = 0, total = 0;
    for (size_t i = 0; i < P->up.size(); ++i) {
        need0 += P->up[i][0];
        total += P->up[i][K - 1];
    }
    P->useful = total > 0 && need0 * 10 <= total * 6 && P->fin[K / 2] * 10 >= static_cast<long long>(output_size) * 2;
    return P;
}

int range_align(const KernelPlan& kp) { return kp.family == Family::Macro ? kp.G : 32; }

// Device action with the zeroing of y fused into the compute (schedules with
// FEMGPU_FLAG_FUSED_ZERO on large outputs; otherwise [memset y, one launch]).  The y memset is an HBM-bound
// pass over the whole output (8 B/row: 17 us of a 179 us P3 2D step) in front of FP64-bound
// kernels.  The cells are split into K slabs (zero_plan: K from the schedule, default 8,
// fewer when a slab would hold less than one wave of CTAs); only the y rows slabs 0 and 1 can
// reach are memset in front; slab k clears the rows slab k+2 reaches first ([zero_hi[k+1],
// zero_hi[k+2])) in a prologue of its own CTAs (kZeroPrologue: a few 8-byte stores per thread,
// free beside the FP64 work).  Slabs alternate between the caller's stream and a worker stream so
// slab k+1's CTAs fill the SMs slab k's tail leaves idle (measured +2.7 us for 4 slabs vs +11 us
// on one stream).  Ordering: slab j needs slabs 0..j-2 complete (they cleared its rows): those on
// its own stream by stream order, those on the other stream through an event on slab j-3.
// Concurrent slabs only RED into y (order-independent up to floating-point reassociation, as
// within one launch), and no slab writes rows another concurrent slab clears (prefix maxima).
// A side-stream memset instead of the fused prologue was measured slower than no overlap:
// memset CTAs take whole CTA slots beside 255-register action CTAs (profiles/r01_zero_overlap.txt).
bool overlapped_zero_action(Instance& I, const KernelPlan& plan, double* d_y, cudaStream_t stream,
                            cudaEvent_t after_zero) {
    // per schedule (FEMGPU_FLAG_FUSED_ZERO, chosen by the tuner where it measures faster);
    // FEMGPU_ZERO_OVERLAP=0 / 1 forces it off / on for every cell-range schedule
    const char* env = std::getenv("FEMGPU_ZERO_OVERLAP");
    const bool on = env ? std::strcmp(env, "0") != 0 : plan.zfused;
    if (!on || !supports_cell_range(plan)) return false;
    // the prologue is compiled only into zfused kernels (it costs up to 7 % elsewhere: C5-adv-P2)
    KernelPlan kp = plan;
    kp.zfused = true;
    if (static_cast<long long>(I.output_size) < kZeroOverlapMinRows || I.cells < kZeroOverlapMinCells) return false;
    // cells one full wave of resident CTAs processes: slabs smaller than that under-fill the GPU
    auto mod = I.module_for(kp);
    const long long cells_per_cta = kp.family == Family::Dmma ? static_cast<long long>(kp.block / 32) * kp.Nc
                                                              : static_cast<long long>(kp.block / std::max(1, kp.msplit)) * std::max(1, kp.G);
    const long long wave = static_cast<long long>(mod->sms) * std::max(1, mod->occupancy) * cells_per_cta;
    const PipePlan& Z = I.zero_plan(range_align(kp), kp.zslabs,
                                    static_cast<int>(std::min<long long>(64, I.cells / std::max(1LL, wave))));
    const int K = static_cast<int>(Z.cb.size()) - 1;
    if (K < 4 || Z.zero_hi[1] * 10 > static_cast<long long>(I.output_size) * 6) return false;  // no locality
    if (!I.s_work) FG_CUDA(cudaStreamCreateWithFlags(&I.s_work, cudaStreamNonBlocking));
    while (static_cast<int>(I.ev_zero.size()) < K + 2) {
        cudaEvent_t e;
        FG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        I.ev_zero.push_back(e);
    }
    // ev_zero[k]: slab k done (on its stream); ev_zero[K]: rows of slabs 0, 1 zeroed
    FG_CUDA(cudaMemsetAsync(d_y, 0, sizeof(double) * static_cast<size_t>(Z.zero_hi[1]), stream));
    if (after_zero) FG_CUDA(cudaEventRecord(after_zero, stream));
    FG_CUDA(cudaEventRecord(I.ev_zero[K], stream));
    FG_CUDA(cudaStreamWaitEvent(I.s_work, I.ev_zero[K], 0));
    for (int k = 0; k < K; ++k) {
        cudaStream_t s = (k & 1) ? I.s_work : stream;
        if (k >= 3) FG_CUDA(cudaStreamWaitEvent(s, I.ev_zero[k - 3], 0));
        double* zp = nullptr;
        long long zn = 0;
        if (k + 2 < K) {
            zp = d_y + Z.zero_hi[k + 1];
            zn = Z.zero_hi[k + 2] - Z.zero_hi[k + 1];
        }
        run_action_range(I, kp, d_y, s, Z.cb[k], Z.cb[k + 1], false, nullptr, zp, zn);
        FG_CUDA(cudaEventRecord(I.ev_zero[k], s));
    }
    // join: the worker stream's last slab (the caller's stream already follows its own slabs)
    FG_CUDA(cudaStreamWaitEvent(stream, I.ev_zero[(K - 1) & 1 ? K - 1 : K - 2], 0));
    I.last_launches = K;
    return true;
}

bool pipelined_host_action(Instance& I, const KernelPlan& kp, const double* const* scalar_inputs,
                           const double* const* vector_inputs, double* y_host, int buf, double* y_dev) {
    double* const Y = y_dev ? y_dev : I.d_y;
    const char* env = std::getenv("FEMGPU_PIPELINE");
    if ((env && std::strcmp(env, "0") == 0) || I.cells < kPipeMinCells || !supports_cell_range(kp)) return false;
    const PipePlan& P = buf < 0 ? I.pipe_plan(range_align(kp)) : I.stream_plan(range_align(kp));
    if (!P.useful) return false;
    const int K = static_cast<int>(P.cb.size()) - 1;
    if (!I.s_h2d) {
        FG_CUDA(cudaStreamCreateWithFlags(&I.s_h2d, cudaStreamNonBlocking));
        FG_CUDA(cudaStreamCreateWithFlags(&I.s_d2h, cudaStreamNonBlocking));
    }
    while (static_cast<int>(I.ev_pipe.size()) < 2 * K + 1) {
        cudaEvent_t e;
        FG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        I.ev_pipe.push_back(e);
    }
    const int d = I.sig.dim;
    if (buf < 0) {
        // previous work on the instance stream (an earlier action) must finish before inputs change
        FG_CUDA(cudaEventRecord(I.ev_pipe[2 * K], I.stream));
        FG_CUDA(cudaStreamWaitEvent(I.s_h2d, I.ev_pipe[2 * K], 0));
    } else {
        // streaming step: this buffer set's inputs were last read by the compute two steps ago and
        // its output last read by that step's download; the other set's step may still be running
        for (int b = 0; b < 2; ++b)
            if (!I.ev_async_comp[b]) {
                FG_CUDA(cudaEventCreateWithFlags(&I.ev_async_comp[b], cudaEventDisableTiming));
                FG_CUDA(cudaEventCreateWithFlags(&I.ev_async_d2h[b], cudaEventDisableTiming));
            }
        if (I.async_used[buf]) {
            FG_CUDA(cudaStreamWaitEvent(I.s_h2d, I.ev_async_comp[buf], 0));
            FG_CUDA(cudaStreamWaitEvent(I.stream, I.ev_async_d2h[buf], 0));
        }
    }
    std::vector<long long> done(P.up.size(), 0);
    long long zeroed = 0, sent = 0;
    // FEMGPU_PIPE_TRACE=1: timing events after every H2D chunk, slab kernel and D2H chunk, printed to
    // stderr as a timeline (us from the start of the action) -- a measurement aid, off by default
    const bool trace = std::getenv("FEMGPU_PIPE_TRACE") != nullptr;
    // (trace experiments: FEMGPU_PIPE_TRACE_SKIP=copies|kernels drops one side -- wrong results)
    const char* skip = std::getenv("FEMGPU_PIPE_TRACE_SKIP");
    const bool no_copy = trace && skip && std::strcmp(skip, "copies") == 0;
    const bool no_kernel = trace && skip && std::strcmp(skip, "kernels") == 0;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        FG_CUDA(cudaEventCreate(&e));
        FG_CUDA(cudaEventRecord(e, st));
        tev.push_back(e);
    };
    mark(I.s_h2d);
    for (int k = 0; k < K; ++k) {
        // H2D: every trial space up to what slab k reads
        for (size_t i = 0; i < I.sspaces.size(); ++i) {
            const long long a = done[i], b = P.up[i][k];
            if (b > a) {
                if (!scalar_inputs || !scalar_inputs[i]) invalid("instance: scalar input length mismatch");
                if (!no_copy) FG_CUDA(cudaMemcpyAsync(I.sspaces[i].d_x + a, scalar_inputs[i] + a, sizeof(double) * (b - a),
                                        cudaMemcpyHostToDevice, I.s_h2d));
                done[i] = b;
            }
        }
        for (size_t i = 0; i < I.vspaces.size(); ++i) {
            const size_t j = I.sspaces.size() + i;
            const long long a = done[j], b = P.up[j][k];
            if (b > a) {
                if (!vector_inputs || !vector_inputs[i]) invalid("instance: vector input length mismatch");
                const int vs = vec_stride(d);
                upload_padded(I.vspaces[i].d_x + a * vs, vector_inputs[i] + a * d, b - a, d,
                              I.vspaces[i].d_stage ? I.vspaces[i].d_stage + a * d : nullptr, I.s_h2d);
                done[j] = b;
            }
        }
        mark(I.s_h2d);
        FG_CUDA(cudaEventRecord(I.ev_pipe[k], I.s_h2d));
        // compute: zero the y rows slab k can newly reach, then the slab
        FG_CUDA(cudaStreamWaitEvent(I.stream, I.ev_pipe[k], 0));
        if (P.zero_hi[k] > zeroed) {
            FG_CUDA(cudaMemsetAsync(Y + zeroed, 0, sizeof(double) * (P.zero_hi[k] - zeroed), I.stream));
            zeroed = P.zero_hi[k];
        }
        if (!no_kernel) run_action_range(I, kp, Y, I.stream, P.cb[k], P.cb[k + 1], false);
        mark(I.stream);
        FG_CUDA(cudaEventRecord(I.ev_pipe[K + k], I.stream));
        // D2H: the rows no later slab touches
        FG_CUDA(cudaStreamWaitEvent(I.s_d2h, I.ev_pipe[K + k], 0));
        if (P.fin[k] > sent) {
            if (!no_copy) FG_CUDA(cudaMemcpyAsync(y_host + sent, Y + sent, sizeof(double) * (P.fin[k] - sent),
                                    cudaMemcpyDeviceToHost, I.s_d2h));
            sent = P.fin[k];
        }
        mark(I.s_d2h);
    }
    if (buf >= 0) {
        FG_CUDA(cudaEventRecord(I.ev_async_comp[buf], I.stream));
        FG_CUDA(cudaEventRecord(I.ev_async_d2h[buf], I.s_d2h));
        I.async_used[buf] = true;
    } else {
        FG_CUDA(cudaEventRecord(I.ev_pipe[2 * K], I.s_d2h));
        FG_CUDA(cudaStreamWaitEvent(I.stream, I.ev_pipe[2 * K], 0));
    }
    if (trace) {
        FG_CUDA(cudaStreamSynchronize(I.stream));
        std::fprintf(stderr, "pipe trace K=%d (us: h2d done, kernel done, d2h done per slab)\n", K);
        for (int k = 0; k < K; ++k) {
            float t[3];
            for (int j = 0; j < 3; ++j) FG_CUDA(cudaEventElapsedTime(&t[j], tev[0], tev[1 + 3 * k + j]));
            std::fprintf(stderr, "  slab %2d: %8.1f %8.1f %8.1f\n", k, t[0] * 1e3, t[1] * 1e3, t[2] * 1e3);
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    I.last_launches = K;
    return true;
}

}  // namespace femgpu
