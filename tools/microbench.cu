// microbench.cu — measures the FP64 denominators of the roofline on this B200
// (MEASURED_PEAKS.json carries only HBM copy and bf16 GEMM figures):
//   dfma   : FP64 FMA pipe, 8 independent chains per thread, full-chip grid
//   dmma   : legacy FP64 tensor path, mma.sync m8n8k4 (SASS DMMA), 4 chains per warp
//   red    : red.global.add.f64 throughput, spread addresses (scatter cost model)
// Prints one JSON object.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[blockIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
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

// even warps DFMA, odd warps DMMA: do the two FP64 paths overlap?
__global__ void mixed_kernel(double* out, int iters) {
    const int warp = threadIdx.x / 32;
    if (warp % 2 == 0) {
        double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
        const double a = 1.0000001, b = 1e-9;
        for (int i = 0; i < iters * 2; ++i) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            }
        }
        double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
        if (s == 12345.678) out[blockIdx.x] = s;
    } else {
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
}

__global__ void red_kernel(double* y, const int* idx, int n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
            atomicAdd(&y[idx[i]], 1.0);
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    double* out;
    CK(cudaMalloc(&out, 1 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // DFMA
    const int blocks = sms * 8, threads = 256, iters = 2048;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    double best_dfma = 0;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
        best_dfma = fl / (ms * 1e-3) > best_dfma ? fl / (ms * 1e-3) : best_dfma;
    }
    // DMMA: 8x8x4 = 256 FMA = 512 flop per warp instruction
    const int mblocks = sms * 8, mthreads = 256, miters = 1024;
    dmma_kernel<<<mblocks, mthreads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    double best_dmma = 0;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        dmma_kernel<<<mblocks, mthreads>>>(out, miters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 512.0 * (mblocks * mthreads / 32) * (double)miters * 8 * 4;
        best_dmma = fl / (ms * 1e-3) > best_dmma ? fl / (ms * 1e-3) : best_dmma;
    }
    // mixed: half the warps DFMA (2*miters x 16 x 8 FMA/thread), half DMMA
    double best_mixed = 0, mixed_ms = 1e30;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        mixed_kernel<<<mblocks, mthreads>>>(out, miters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double warps = mblocks * mthreads / 32.0;
        double fl = 0.5 * warps * (512.0 * miters * 8 * 4) + 0.5 * warps * 32 * (2.0 * 2 * miters * 16 * 8);
        if (fl / (ms * 1e-3) > best_mixed) { best_mixed = fl / (ms * 1e-3); mixed_ms = ms; }
    }
    // RED f64: 64M atomics over 16M distinct addresses (pseudo-random permutation-ish)
    const int n = 1 << 26, m = 1 << 24;
    int* idx;
    double* y;
    CK(cudaMalloc(&idx, sizeof(int) * n));
    CK(cudaMalloc(&y, sizeof(double) * m));
    int* h = (int*)malloc(sizeof(int) * n);
    unsigned s = 12345;
    for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = (int)((s >> 7) % m); }
    CK(cudaMemcpy(idx, h, sizeof(int) * n, cudaMemcpyHostToDevice));
    red_kernel<<<sms * 8, 256>>>(y, idx, n, 1);
    CK(cudaDeviceSynchronize());
    double best_red = 0;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        red_kernel<<<sms * 8, 256>>>(y, idx, n, 1);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        best_red = n / (ms * 1e-3) > best_red ? n / (ms * 1e-3) : best_red;
    }
    // RED with locality: sequential addresses, 8 atomics per address from consecutive threads
    for (int i = 0; i < n; ++i) h[i] = (i / 8) % m;
    CK(cudaMemcpy(idx, h, sizeof(int) * n, cudaMemcpyHostToDevice));
    double best_red_local = 0;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        red_kernel<<<sms * 8, 256>>>(y, idx, n, 1);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        best_red_local = n / (ms * 1e-3) > best_red_local ? n / (ms * 1e-3) : best_red_local;
    }
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, "
           "\"mixed_dfma_dmma_tflops\": %.3f, \"red_f64_random_gops\": %.2f, \"red_f64_local8_gops\": %.2f, \"how\": \"best of 5 (3), CUDA events; "
           "dfma 8 chains x %d thr x %d blk; dmma m8n8k4 4 chains; red 64M adds over 16M addresses\"}\n",
           prop.name, sms, best_dfma / 1e12, best_dmma / 1e12, best_mixed / 1e12, best_red / 1e9, best_red_local / 1e9, threads, blocks);
    return 0;
}
