// peaks.cu — ahead-of-time sm_100a kernels of libfemgpu: the FP64 roofline denominators.
// MEASURED_PEAKS.json (driver-written) carries only an HBM copy and a bf16 GEMM figure, so
// the FP64 peaks are measured live on the same GPU: femgpu_fp64_peak (DFMA: 8 independent
// FMA chains per thread, 8 CTAs of 256 threads per SM) and femgpu_fp64_dmma_peak (DMMA
// m8n8k4: 4 accumulators per warp), each the best of 5 timed with CUDA events.  The form
// roofline uses the larger of the two (the machine's FP64 peak).
#include <cuda_runtime.h>

#include "femgpu_internal.hpp"

namespace {

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[blockIdx.x] = s;
}

// FP64 tensor path: mma.sync m8n8k4 .f64 (SASS DMMA), 4 independent accumulators per warp.
__global__ void dmma_peak_kernel(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
        }
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

}  // namespace

extern "C" femgpu_status femgpu_fp64_dmma_peak(double* tflops) {
    try {
        int dev = 0, sms = 0;
        FG_CUDA(cudaGetDevice(&dev));
        FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        double* out = nullptr;
        FG_CUDA(cudaMalloc(&out, sizeof(double) * 8 * sms));
        cudaEvent_t e0, e1;
        FG_CUDA(cudaEventCreate(&e0));
        FG_CUDA(cudaEventCreate(&e1));
        const int blocks = 8 * sms, threads = 256, iters = 1024;
        dmma_peak_kernel<<<blocks, threads>>>(out, 16);
        FG_CUDA(cudaGetLastError());
        double best = 0.0;
        for (int t = 0; t < 5; ++t) {
            FG_CUDA(cudaEventRecord(e0));
            dmma_peak_kernel<<<blocks, threads>>>(out, iters);
            FG_CUDA(cudaEventRecord(e1));
            FG_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            FG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            const double flops = 512.0 * (blocks * threads / 32) * static_cast<double>(iters) * 8 * 4;
            if (flops / (ms * 1e-3) > best) best = flops / (ms * 1e-3);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        if (tflops) *tflops = best / 1e12;
        return FEMGPU_OK;
    } catch (const femgpu::Error& e) {
        return e.code;
    }
}

extern "C" femgpu_status femgpu_fp64_peak(double* tflops, double* sm_clock_ghz) {
    try {
        int dev = 0, sms = 0, clk_khz = 0;
        FG_CUDA(cudaGetDevice(&dev));
        FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
        double* out = nullptr;
        FG_CUDA(cudaMalloc(&out, sizeof(double) * 8 * sms));
        cudaEvent_t e0, e1;
        FG_CUDA(cudaEventCreate(&e0));
        FG_CUDA(cudaEventCreate(&e1));
        const int blocks = 8 * sms, threads = 256, iters = 2048;
        dfma_peak_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
        FG_CUDA(cudaGetLastError());
        double best = 0.0;
        for (int t = 0; t < 5; ++t) {
            FG_CUDA(cudaEventRecord(e0));
            dfma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
            FG_CUDA(cudaEventRecord(e1));
            FG_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            FG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            const double flops = 2.0 * blocks * threads * static_cast<double>(iters) * 16 * 8;
            if (flops / (ms * 1e-3) > best) best = flops / (ms * 1e-3);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        if (tflops) *tflops = best / 1e12;
        if (sm_clock_ghz) *sm_clock_ghz = clk_khz / 1e6;
        return FEMGPU_OK;
    } catch (const femgpu::Error& e) {
        return e.code;
    }
}
