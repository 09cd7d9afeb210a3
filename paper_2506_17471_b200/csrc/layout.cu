// layout.cu — ahead-of-time sm_100a kernel of libfemgpu: re-blocks node-major [node][dim]
// host data (vector inputs, coordinates) into the padded device layout [node][vec_stride(dim)]
// (femgpu_internal.hpp).  The host array is copied contiguously (one DMA) into a staging buffer
// and padded on the device: a pitched cudaMemcpy2D with 24-byte rows would issue one tiny
// transfer per node.
#include <cuda_runtime.h>

#include "femgpu_internal.hpp"

namespace {

__global__ void pad_rows_kernel(const double* __restrict__ src, double* __restrict__ dst, long long n, int d, int vs) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        for (int c = 0; c < vs; ++c) dst[i * vs + c] = c < d ? src[i * d + c] : 0.0;
    }
}

}  // namespace

namespace femgpu {

void upload_padded(double* dst, const double* src_host, long long rows, int d, double* staging, cudaStream_t stream) {
    const int vs = vec_stride(d);
    if (vs == d) {
        FG_CUDA(cudaMemcpyAsync(dst, src_host, sizeof(double) * rows * d, cudaMemcpyHostToDevice, stream));
        return;
    }
    FG_CUDA(cudaMemcpyAsync(staging, src_host, sizeof(double) * rows * d, cudaMemcpyHostToDevice, stream));
    const long long blocks = std::min<long long>((rows + 255) / 256, 148LL * 16);
    if (rows > 0) pad_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(staging, dst, rows, d, vs);
    FG_CUDA(cudaGetLastError());
}

}  // namespace femgpu
