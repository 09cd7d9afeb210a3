// devspec_bench.cu — measures the saturation points of the reference's DeviceSpec
// (perf_model.hpp:21-31) on this B200: global (HBM) read bandwidth and shared-memory bandwidth as
// a function of resident sub-groups (warps) per SM, one CTA per SM, persistent grid of 148 CTAs.
// saturation_subgroups_* = the smallest warp count reaching 90 % of the best bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/devspec_bench tools/devspec_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void hbm_read(const double2* __restrict__ x, long long n, double* out) {
    double2 acc = make_double2(0, 0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(x + i);
        acc.x += v.x;
        acc.y += v.y;
    }
    if (acc.x == 1.2345) out[0] = acc.y;
}

__global__ void smem_read(double* out, int iters) {
    __shared__ double2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, -i);
    __syncthreads();
    double2 acc = make_double2(0, 0);
    int k = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double2 v = s[(k + u * 32) & 2047];
            acc.x += v.x;
            acc.y += v.y;
        }
        k = (k + 256) & 2047;
    }
    if (acc.x == 1.2345) out[0] = acc.y;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1LL << 28;  // 4 GiB of double2
    double2* x;
    double* out;
    cudaMalloc(&x, n * sizeof(double2));
    cudaMemset(x, 0, n * sizeof(double2));
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int warps[] = {1, 2, 4, 8, 12, 16, 24, 32};
    double hbm[8], sm[8];
    for (int w = 0; w < 8; ++w) {
        float ms;
        hbm_read<<<sms, 32 * warps[w]>>>(x, n, out);
        cudaEventRecord(e0);
        hbm_read<<<sms, 32 * warps[w]>>>(x, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        hbm[w] = n * sizeof(double2) / (ms * 1e-3) / 1e9;
        const int iters = 4096;
        smem_read<<<sms, 32 * warps[w]>>>(out, 16);
        cudaEventRecord(e0);
        smem_read<<<sms, 32 * warps[w]>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        sm[w] = (double)sms * 32 * warps[w] * iters * 8 * sizeof(double2) / (ms * 1e-3) / 1e9;
    }
    double hb = 0, sb = 0;
    for (int w = 0; w < 8; ++w) { hb = hbm[w] > hb ? hbm[w] : hb; sb = sm[w] > sb ? sm[w] : sb; }
    int hs = 0, ss = 0;
    for (int w = 7; w >= 0; --w) { if (hbm[w] >= 0.9 * hb) hs = warps[w]; if (sm[w] >= 0.9 * sb) ss = warps[w]; }
    printf("{\"sms\": %d, \"warps_per_sm\": [", sms);
    for (int w = 0; w < 8; ++w) printf("%s%d", w ? ", " : "", warps[w]);
    printf("], \"hbm_read_gbs\": [");
    for (int w = 0; w < 8; ++w) printf("%s%.1f", w ? ", " : "", hbm[w]);
    printf("], \"smem_read_gbs\": [");
    for (int w = 0; w < 8; ++w) printf("%s%.1f", w ? ", " : "", sm[w]);
    printf("], \"saturation_subgroups_global\": %d, \"saturation_subgroups_local\": %d, \"peak_local_bw_gbs\": %.0f}\n", hs, ss, sb);
    return 0;
}
