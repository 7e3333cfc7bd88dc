// nvlink_probe.cu -- standalone NVLink probe (2 GPUs, one process, P2P):
// pull (load-based) vs push (store-based) two-shot mean of a 400 MB buffer,
// plus raw one-way read / write / copy rates. Tooling, not product code.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/nvlink_probe tools/nvlink_probe.cu
//   ./tools/nvlink_probe [n_floats]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void copy_k(float4* __restrict__ dst, const float4* __restrict__ src, long n) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x, s = (long)gridDim.x * blockDim.x;
    for (; i + 3 * s < n; i += 4 * s) {
        float4 a = __ldcg(src + i), b = __ldcg(src + i + s), c = __ldcg(src + i + 2 * s), d = __ldcg(src + i + 3 * s);
        __stcg(dst + i, a); __stcg(dst + i + s, b); __stcg(dst + i + 2 * s, c); __stcg(dst + i + 3 * s, d);
    }
    for (; i < n; i += s) __stcg(dst + i, __ldcg(src + i));
}

__device__ __forceinline__ float4 add4(float4 a, float4 b, float k) {
    return make_float4((a.x + b.x) * k, (a.y + b.y) * k, (a.z + b.z) * k, (a.w + b.w) * k);
}

// pull two-shot over shard [v0, v0+nv): read local + remote, write both
__global__ void pull_k(float4* loc, float4* rem, long v0, long nv) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x, s = (long)gridDim.x * blockDim.x;
    for (; i + 3 * s < nv; i += 4 * s) {
        float4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = __ldcg(loc + v0 + i + u * s); b[u] = __ldcg(rem + v0 + i + u * s); }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float4 r = add4(a[u], b[u], 0.5f);
            __stcg(loc + v0 + i + u * s, r); __stcg(rem + v0 + i + u * s, r);
        }
    }
    for (; i < nv; i += s) {
        float4 r = add4(__ldcg(loc + v0 + i), __ldcg(rem + v0 + i), 0.5f);
        __stcg(loc + v0 + i, r); __stcg(rem + v0 + i, r);
    }
}

// push phase 2: owner sums its copy and the peer's pushed copy (local scratch), writes both
__global__ void push2_k(float4* loc, const float4* scratch, float4* rem, long v0, long nv) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x, s = (long)gridDim.x * blockDim.x;
    for (; i + 3 * s < nv; i += 4 * s) {
        float4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { a[u] = __ldcg(loc + v0 + i + u * s); b[u] = __ldcg(scratch + i + u * s); }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float4 r = add4(a[u], b[u], 0.5f);
            __stcg(loc + v0 + i + u * s, r); __stcg(rem + v0 + i + u * s, r);
        }
    }
    for (; i < nv; i += s) {
        float4 r = add4(__ldcg(loc + v0 + i), __ldcg(scratch + i), 0.5f);
        __stcg(loc + v0 + i, r); __stcg(rem + v0 + i, r);
    }
}

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 100000000L;
    long nv = n / 4, half = nv / 2;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float4 *buf[2], *scr[2];
    cudaStream_t st[2];
    for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaDeviceEnablePeerAccess(1 - d, 0));
        CK(cudaMalloc(&buf[d], nv * 16));
        CK(cudaMalloc(&scr[d], half * 16 + 16));
        CK(cudaMemset(buf[d], 0, nv * 16));
        CK(cudaMemset(scr[d], 0, half * 16));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    }
    auto sync_all = [&]() { for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaStreamSynchronize(st[d])); } };
    auto bench = [&](const char* name, double bytes_per_dir, std::function<void(int)> body) {
        for (int it = 0; it < 3; ++it) body(it);
        sync_all();
        const int iters = 20;
        auto t0 = std::chrono::high_resolution_clock::now();
        for (int it = 0; it < iters; ++it) body(it);
        sync_all();
        double us = std::chrono::duration<double, std::micro>(std::chrono::high_resolution_clock::now() - t0).count() / iters;
        printf("%-44s %9.1f us  %7.1f GB/s per direction\n", name, us, bytes_per_dir / us * 1e-3);
    };
    for (int blocks_per_sm : {2, 4, 8}) {
        const int grid = sms * blocks_per_sm, thr = 256;
        printf("--- grid %d x %d\n", grid, thr);
        const double S = nv * 16.0;
        // raw: each GPU reads the peer's half (one direction per GPU: both directions busy)
        bench("read  peer half -> local (both GPUs)", S / 2, [&](int) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); copy_k<<<grid, thr, 0, st[d]>>>(scr[d], buf[1 - d], half); }
        });
        bench("write local half -> peer (both GPUs)", S / 2, [&](int) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); copy_k<<<grid, thr, 0, st[d]>>>(scr[1 - d], buf[d], half); }
        });
        bench("read  peer half, one GPU only", S / 2, [&](int) {
            CK(cudaSetDevice(0)); copy_k<<<grid, thr, 0, st[0]>>>(scr[0], buf[1], half);
        });
        bench("write local half, one GPU only", S / 2, [&](int) {
            CK(cudaSetDevice(0)); copy_k<<<grid, thr, 0, st[0]>>>(scr[1], buf[0], half);
        });
        // pull two-shot mean: rank d owns half d
        bench("mean pull two-shot (current)", S, [&](int) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); pull_k<<<grid, thr, 0, st[d]>>>(buf[d], buf[1 - d], d * half, half); }
        });
        // push two-shot: phase 1 each pushes the peer-owned half into the peer's scratch; phase 2 owner sums + pushes
        cudaEvent_t ev[2];
        for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventCreateWithFlags(&ev[d], cudaEventDisableTiming)); }
        bench("mean push two-shot (stores only)", S, [&](int) {
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                copy_k<<<grid, thr, 0, st[d]>>>(scr[1 - d], buf[d] + (1 - d) * half, half);
                CK(cudaEventRecord(ev[d], st[d]));
            }
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaStreamWaitEvent(st[d], ev[1 - d], 0));
                push2_k<<<grid, thr, 0, st[d]>>>(buf[d], scr[d], buf[1 - d], d * half, half);
            }
        });
        bench("push phase 1 only (both)", S / 2, [&](int) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); copy_k<<<grid, thr, 0, st[d]>>>(scr[1 - d], buf[d] + (1 - d) * half, half); }
        });
        bench("push phase 2 only (both)", S / 2, [&](int) {
            for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); push2_k<<<grid, thr, 0, st[d]>>>(buf[d], scr[d], buf[1 - d], d * half, half); }
        });
        for (int d = 0; d < 2; ++d) { CK(cudaSetDevice(d)); CK(cudaEventDestroy(ev[d])); }
    }
    return 0;
}
