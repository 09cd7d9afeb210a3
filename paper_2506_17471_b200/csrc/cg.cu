// cg.cu — the action's caller on the device: conjugate gradients for a symmetric
// positive-definite operator, entirely on the instance stream.
//
// Per iteration: one output-pipelined action A p (the next iteration's output buffer is zeroed inside
// the same launch), one fused update kernel (x += alpha p, r -= alpha A p, block partials of r.r),
// one fused direction kernel (p = r + beta p), and fixed-order reductions.  The scalars alpha, beta,
// r.r and p.Ap stay in device memory: no host round trip except the residual check every
// `check_every` iterations (between checks, pairs of iterations replay as a CUDA graph).  Reductions use a fixed grid and fixed in-block order (no floating-point
// atomics); the action's red.add scatter is the only order-dependent step (colour scatter, SCATTER_COLOR,
// makes it bitwise reproducible too).
#include <cmath>
#include <cuda_runtime.h>

#include "femgpu_internal.hpp"

namespace {

constexpr int kBlocks = 1184;  // 8 CTAs per SM (streaming needs the parallelism); every reduction has the same partial layout
constexpr int kThreads = 256;

__device__ __forceinline__ void block_sum_to(double v, double* out) {
    __shared__ double red[kThreads];
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// part[block] = sum over this block's grid-stride elements of a[i] * b[i]
__global__ void dot_partial(const double* __restrict__ a, const double* __restrict__ b, long long n, double* part) {
    double s = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n; i += static_cast<long long>(kBlocks) * kThreads)
        s += a[i] * b[i];
    block_sum_to(s, part + blockIdx.x);
}

// *out = sum of the kBlocks partials (one block, fixed order)
__global__ void dot_final(const double* __restrict__ part, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < kBlocks; i += kThreads) s += part[i];
    block_sum_to(s, out);
}

// alpha = rr / pap; x += alpha p; r -= alpha ap; partials of r.r
__global__ void update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                          const double* __restrict__ ap, long long n, const double* rr, const double* pap, double* part) {
    const double alpha = *rr / *pap;
    double s = 0.0;
    for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n; i += static_cast<long long>(kBlocks) * kThreads) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        s += ri * ri;
    }
    block_sum_to(s, part + blockIdx.x);
}

// beta = rr_new / rr_old; p = r + beta p
__global__ void update_p(double* __restrict__ p, const double* __restrict__ r, long long n, const double* rr_new,
                         const double* rr_old) {
    const double beta = *rr_new / *rr_old;
    for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n; i += static_cast<long long>(kBlocks) * kThreads)
        p[i] = r[i] + beta * p[i];
}

// r = b - ax (ax may be null: r = b); p = r
__global__ void init_rp(double* __restrict__ r, double* __restrict__ p, const double* __restrict__ b, const double* ax, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; i < n; i += static_cast<long long>(kBlocks) * kThreads) {
        const double ri = ax ? b[i] - ax[i] : b[i];
        r[i] = ri;
        p[i] = ri;
    }
}

}  // namespace

namespace femgpu {

// y = A v with the instance's scalar trial space 0 reading v (pointer swapped in for the launch)
static void apply_into(Instance& I, const KernelPlan& kp, double* v, double* y, double* y_next, cudaStream_t s) {
    std::swap(I.sspaces[0].d_x, v);
    try {
        run_action_pipelined(I, kp, y, y_next, s);
    } catch (...) {
        std::swap(I.sspaces[0].d_x, v);
        throw;
    }
    std::swap(I.sspaces[0].d_x, v);
}

void device_cg(Instance& I, const KernelPlan& kp, const double* b, double* x, double rtol, int maxiter, int check_every,
               int* iterations, double* rel_residual) {
    if (I.sspaces.size() != 1 || !I.vspaces.empty())
        invalid("cg: one scalar trial space required (a square scalar operator)");
    const long long n = I.output_size;
    if (I.sspaces[0].global != n) invalid("cg: square operators only (trial and test sizes differ)");
    if (check_every < 1) check_every = 1;
    cudaStream_t s = I.stream;
    if (I.cg_work.empty()) {
        for (int k = 0; k < 4; ++k) I.cg_work.push_back(I.alloc<double>(static_cast<size_t>(n)));  // r, p, ap[2]
        I.cg_work.push_back(I.alloc<double>(kBlocks + 8));                                    // partials + scalars
    }
    double *r = I.cg_work[0], *p = I.cg_work[1], *ap[2] = {I.cg_work[2], I.cg_work[3]};
    double* part = I.cg_work[4];
    double* sc = part + kBlocks;  // sc[0], sc[1]: r.r (alternating), sc[2]: p.Ap, sc[3]: b.b
    const dim3 g(kBlocks), t(kThreads);
    // r = b - A x, p = r
    FG_CUDA(cudaMemsetAsync(ap[0], 0, sizeof(double) * static_cast<size_t>(n), s));
    apply_into(I, kp, x, ap[0], ap[1], s);
    init_rp<<<g, t, 0, s>>>(r, p, b, ap[0], n);
    dot_partial<<<g, t, 0, s>>>(b, b, n, part);
    dot_final<<<1, t, 0, s>>>(part, sc + 3);
    dot_partial<<<g, t, 0, s>>>(r, r, n, part);
    dot_final<<<1, t, 0, s>>>(part, sc + 0);
    FG_CUDA(cudaGetLastError());
    double host[4];
    FG_CUDA(cudaMemcpyAsync(host, sc, sizeof host, cudaMemcpyDeviceToHost, s));
    FG_CUDA(cudaStreamSynchronize(s));
    const double bnorm = std::sqrt(host[3]);
    double res = std::sqrt(host[0]);
    int it = 0, cur = 0, a = 1;  // r.r in sc[cur]; ap[a] is zero on entry (zeroed by the first action)
    auto iteration = [&]() {
        apply_into(I, kp, p, ap[a], ap[a ^ 1], s);  // ap[a] = A p, ap[a ^ 1] zeroed for the next iteration
        dot_partial<<<g, t, 0, s>>>(p, ap[a], n, part);
        dot_final<<<1, t, 0, s>>>(part, sc + 2);
        update_xr<<<g, t, 0, s>>>(x, r, p, ap[a], n, sc + cur, sc + 2, part);
        dot_final<<<1, t, 0, s>>>(part, sc + (cur ^ 1));
        update_p<<<g, t, 0, s>>>(p, r, n, sc + (cur ^ 1), sc + cur);
        FG_CUDA(cudaGetLastError());
        cur ^= 1;
        a ^= 1;
    };
    // Between residual checks the iterations replay as a CUDA graph of two iterations (the buffer
    // roles alternate with period 2): one launch instead of ~14 (small meshes are launch-bound).
    cudaGraphExec_t pair = nullptr;
    if (check_every % 2 == 0 && maxiter >= 2 && res > rtol * bnorm) {
        cudaGraph_t gr = nullptr;
        FG_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            iteration();
            iteration();
        } catch (...) {
            cudaStreamEndCapture(s, &gr);
            if (gr) cudaGraphDestroy(gr);
            throw;
        }
        FG_CUDA(cudaStreamEndCapture(s, &gr));
        FG_CUDA(cudaGraphInstantiate(&pair, gr, 0));
        FG_CUDA(cudaGraphDestroy(gr));
    }
    while (res > rtol * bnorm && it < maxiter) {
        if (pair && it % 2 == 0 && maxiter - it >= 2) {
            FG_CUDA(cudaGraphLaunch(pair, s));  // two iterations; cur and a come back to their values
            it += 2;
        } else {
            iteration();
            ++it;
        }
        if (it % check_every == 0 || it >= maxiter) {
            FG_CUDA(cudaMemcpyAsync(host, sc + cur, sizeof(double), cudaMemcpyDeviceToHost, s));
            FG_CUDA(cudaStreamSynchronize(s));
            res = std::sqrt(host[0]);
            if (!std::isfinite(res)) break;
        }
    }
    if (pair) cudaGraphExecDestroy(pair);
    check_failure(I, kp, s);
    if (iterations) *iterations = it;
    if (rel_residual) *rel_residual = bnorm > 0 ? res / bnorm : res;
}

}  // namespace femgpu
