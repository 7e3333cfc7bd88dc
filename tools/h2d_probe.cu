// h2d_probe.cu -- host-to-device rates of a 400 MB fp32 buffer in pinned host
// memory: SM loads straight from the (UVA-mapped) host pointer. Tooling only.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o tools/_h2d_probe.so tools/h2d_probe.cu
#include <cuda_runtime.h>

__global__ void pull_kernel(float4* __restrict__ dst, const float4* __restrict__ src, long n) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x, s = (long)gridDim.x * blockDim.x;
    for (; i + 3 * s < n; i += 4 * s) {
        float4 a = __ldcs(src + i), b = __ldcs(src + i + s), c = __ldcs(src + i + 2 * s), d = __ldcs(src + i + 3 * s);
        __stcs(dst + i, a); __stcs(dst + i + s, b); __stcs(dst + i + 2 * s, c); __stcs(dst + i + 3 * s, d);
    }
    for (; i < n; i += s) __stcs(dst + i, __ldcs(src + i));
}

extern "C" int pull_launch(void* dst, const void* src, long n_float4, int grid, int block, void* stream) {
    pull_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<float4*>(dst),
                                                                        static_cast<const float4*>(src), n_float4);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
