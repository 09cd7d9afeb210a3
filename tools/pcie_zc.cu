// PCIe duplex experiments for the e2e pipeline: copy engines (cudaMemcpyAsync, chunked) versus SM
// zero-copy kernels over mapped pinned host memory, one direction each or both.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_zc tools/pcie_zc.cu
// usage: ./pcie_zc [chunks] [ctas]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); std::exit(1); } } while (0)

// grid-stride 16-byte copy (src/dst may be mapped host memory)
__global__ void copy16(const double2* __restrict__ src, double2* __restrict__ dst, long long n2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main(int argc, char** argv) {
    const long long n = 9938375LL & ~1LL;  // C2 x / y
    const int K = argc > 1 ? std::atoi(argv[1]) : 8;
    const int ctas = argc > 2 ? std::atoi(argv[2]) : 264;
    double *h_in, *h_out, *d_in, *d_out, *m_in, *m_out;
    CK(cudaHostAlloc(&h_in, n * 8, cudaHostAllocMapped));
    CK(cudaHostAlloc(&h_out, n * 8, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&m_in, h_in, 0));
    CK(cudaHostGetDevicePointer(&m_out, h_out, 0));
    for (long long i = 0; i < n; ++i) h_in[i] = 1.0;
    CK(cudaMalloc(&d_in, n * 8));
    CK(cudaMalloc(&d_out, n * 8));
    cudaStream_t su, sd;
    CK(cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, eu, ed;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&eu)); CK(cudaEventCreate(&ed));
    auto chunk = [&](int k) { return n / K * k & ~1LL; };
    // mode bits: 1 = H2D, 2 = D2H; up/dn: 0 = copy engine, 1 = SM kernel
    auto run = [&](int dirs, int up_sm, int dn_sm) {
        for (int k = 0; k < K; ++k) {
            const long long a = chunk(k), b = k + 1 == K ? n : chunk(k + 1);
            if (dirs & 1) {
                if (up_sm) copy16<<<ctas, 256, 0, su>>>((const double2*)(m_in + a), (double2*)(d_in + a), (b - a) / 2);
                else CK(cudaMemcpyAsync(d_in + a, h_in + a, (b - a) * 8, cudaMemcpyHostToDevice, su));
            }
            if (dirs & 2) {
                if (dn_sm) copy16<<<ctas, 256, 0, sd>>>((const double2*)(d_out + a), (double2*)(m_out + a), (b - a) / 2);
                else CK(cudaMemcpyAsync(h_out + a, d_out + a, (b - a) * 8, cudaMemcpyDeviceToHost, sd));
            }
        }
    };
    auto timed = [&](int dirs, int up_sm, int dn_sm) {
        run(dirs, up_sm, dn_sm);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 10; ++r) {
            CK(cudaEventRecord(e0, su));
            CK(cudaStreamWaitEvent(sd, e0, 0));
            run(dirs, up_sm, dn_sm);
            CK(cudaEventRecord(ed, sd));
            CK(cudaStreamWaitEvent(su, ed, 0));
            CK(cudaEventRecord(e1, su));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        return best;
    };
    std::printf("{\"chunks\": %d, \"ctas\": %d, \"MB_each\": %.1f", K, ctas, n * 8 / 1e6);
    std::printf(", \"h2d_ce\": %.3f, \"h2d_sm\": %.3f", timed(1, 0, 0), timed(1, 1, 0));
    std::printf(", \"d2h_ce\": %.3f, \"d2h_sm\": %.3f", timed(2, 0, 0), timed(2, 0, 1));
    std::printf(", \"both_ce_ce\": %.3f, \"both_sm_ce\": %.3f, \"both_ce_sm\": %.3f, \"both_sm_sm\": %.3f}\n",
                timed(3, 0, 0), timed(3, 1, 0), timed(3, 0, 1), timed(3, 1, 1));
    return 0;
}
