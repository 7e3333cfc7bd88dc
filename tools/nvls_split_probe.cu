// nvls_split_probe.cu -- NVLink mean decomposition probe (tooling, not product
// code). Loaded by tools/nvls_split_probe.py (torchrun, torch symmetric memory
// for the allocation and the peer / multicast addresses). Each rank works on
// its shard [v0, v1) of the float4 vectors of a symmetric fp32 buffer:
//
//   mode 0  NVLS mean          multimem.ld_reduce + multimem.st    (product path)
//   mode 1  ld_reduce only     multimem.ld_reduce, local plain store
//   mode 2  multicast st only  local load, multimem.st
//   mode 3  P2P two-shot       W peer loads, W peer stores          (product path)
//   mode 4  split              first `split_vec` vectors of the shard NVLS,
//                              the rest P2P, blocks divided by `nvls_blocks`
//   mode 5  ld_reduce + P2P st multimem.ld_reduce, W peer stores
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        -o tools/_nvls_split_probe.so tools/nvls_split_probe.cu
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int W = 4;
constexpr int U = 4;

__device__ __forceinline__ float4 ldred(const float* p) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}
__device__ __forceinline__ void mst(float* p, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 sc(float4 v, float s) { return make_float4(v.x * s, v.y * s, v.z * s, v.w * s); }

struct Args {
    float* bufs[8];
    float* mc;
    int rank, world;
    long v0, v1;       // shard (float4 units)
    long split_vec;    // mode 4: NVLS part length
    int nvls_blocks;   // mode 4: blocks on the NVLS part
    int mode;
    float scale;
};

__device__ void nvls_range(const Args& a, long b, long e, long tid, long stride, int mode) {
    float4* loc = reinterpret_cast<float4*>(a.bufs[a.rank]);
    long i = b + tid;
    for (; i + (U - 1) * stride < e; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (mode == 2) v[u] = __ldcg(loc + i + u * stride);
            else v[u] = ldred(a.mc + 4 * (i + u * stride));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (mode == 1) __stcg(loc + i + u * stride, sc(v[u], a.scale));
            else if (mode == 5) {
#pragma unroll
                for (int r = 0; r < W; ++r) __stcg(reinterpret_cast<float4*>(a.bufs[r]) + i + u * stride, sc(v[u], a.scale));
            } else mst(a.mc + 4 * (i + u * stride), sc(v[u], a.scale));
        }
    }
    for (; i < e; i += stride) {
        float4 v = mode == 2 ? __ldcg(loc + i) : ldred(a.mc + 4 * i);
        if (mode == 1) __stcg(loc + i, sc(v, a.scale));
        else if (mode == 5) {
            for (int r = 0; r < W; ++r) __stcg(reinterpret_cast<float4*>(a.bufs[r]) + i, sc(v, a.scale));
        } else mst(a.mc + 4 * i, sc(v, a.scale));
    }
}

__device__ void p2p_range(const Args& a, long b, long e, long tid, long stride) {
    constexpr int UP = 2;
    const float4* src[W];
    float4* dst[W];
#pragma unroll
    for (int r = 0; r < W; ++r) {
        src[r] = reinterpret_cast<const float4*>(a.bufs[r]);
        dst[r] = reinterpret_cast<float4*>(a.bufs[r]);
    }
    long i = b + tid;
    for (; i + (UP - 1) * stride < e; i += UP * stride) {
        float4 v[UP][W];
#pragma unroll
        for (int u = 0; u < UP; ++u)
#pragma unroll
            for (int r = 0; r < W; ++r) v[u][r] = __ldcg(src[r] + i + u * stride);
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            float4 acc = v[u][0];
#pragma unroll
            for (int r = 1; r < W; ++r) {
                acc.x += v[u][r].x; acc.y += v[u][r].y; acc.z += v[u][r].z; acc.w += v[u][r].w;
            }
            acc = sc(acc, a.scale);
#pragma unroll
            for (int r = 0; r < W; ++r) __stcg(dst[r] + i + u * stride, acc);
        }
    }
    for (; i < e; i += stride) {
        float4 acc = __ldcg(src[0] + i);
#pragma unroll
        for (int r = 1; r < W; ++r) {
            float4 v = __ldcg(src[r] + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        acc = sc(acc, a.scale);
#pragma unroll
        for (int r = 0; r < W; ++r) __stcg(dst[r] + i, acc);
    }
}

__global__ void __launch_bounds__(512) probe_kernel(Args a) {
    const long nb = gridDim.x, bid = blockIdx.x;
    if (a.mode == 3) {
        p2p_range(a, a.v0, a.v1, bid * blockDim.x + threadIdx.x, nb * blockDim.x);
    } else if (a.mode == 4) {
        const long vm = a.v0 + a.split_vec;
        if (bid < a.nvls_blocks)
            nvls_range(a, a.v0, vm, bid * blockDim.x + threadIdx.x, (long)a.nvls_blocks * blockDim.x, 0);
        else
            p2p_range(a, vm, a.v1, (bid - a.nvls_blocks) * blockDim.x + threadIdx.x,
                      (nb - a.nvls_blocks) * blockDim.x);
    } else {
        nvls_range(a, a.v0, a.v1, bid * blockDim.x + threadIdx.x, nb * blockDim.x, a.mode);
    }
}

}  // namespace

extern "C" int probe_launch(float* const* bufs, float* mc, int rank, int world, long v0, long v1, long split_vec,
                            int nvls_blocks, int mode, float scale, int grid, int block, void* stream) {
    if (world != W) return 1;
    Args a{};
    for (int r = 0; r < world; ++r) a.bufs[r] = bufs[r];
    a.mc = mc;
    a.rank = rank;
    a.world = world;
    a.v0 = v0;
    a.v1 = v1;
    a.split_vec = split_vec;
    a.nvls_blocks = nvls_blocks;
    a.mode = mode;
    a.scale = scale;
    probe_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
