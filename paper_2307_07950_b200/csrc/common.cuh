// common.cuh -- internal helpers shared by the translation units of
// libselsync_b200.so (not part of the C-ABI; hidden visibility).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

namespace ss_internal {

// record an error message for ss_last_error() and return `code`
int fail(int code, const char* fmt, ...);
// SS_OK or SS_ERR_CUDA with the pending launch error
int check_launch(const char* what);
// multiprocessor count of the current device
int sm_count();
// K13+K2 kernel (fused update + ||g||^2 + signal step) for a prepared step,
// and the float4 vectors per thread and stream its grid is sized for
void* k13_kernel(bool mom, bool nest, int* per_thread);

}  // namespace ss_internal

namespace {

// A block's index within its rank's grid and that grid's size. A launch for
// one rank uses blockIdx.x / gridDim.x; the colocated launch (the grids of
// several ranks sharing one device in ONE cooperative launch) hands each rank
// a contiguous slice of blocks.
struct VBlk {
    int bid;
    int n;
};
__device__ __forceinline__ VBlk hw_blk() {
    return VBlk{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x)};
}

// Programmatic dependent launch. The hot kernels are launched with
// programmatic stream serialization, so their blocks can be placed on SMs
// while the previous kernel in the stream is still draining. Every such kernel
// calls pdl_wait() before it touches memory: it returns once the previous grid
// has completed and its writes are visible. A launch without the attribute
// returns from it at once. pdl_trigger() lets the next launch in the stream
// start being placed; it gives no memory guarantee, so it can run first thing.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// SS_PDL=0 launches without the attribute (A/B knob); read once per process
inline bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("SS_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// Launch `kernel` on a 1-D grid of `threads`-thread blocks with programmatic
// stream serialization (and the cooperative attribute when `coop`).
template <typename... P, typename... A>
cudaError_t launch_ex(void (*kernel)(P...), int grid, int threads, cudaStream_t stream, bool coop, A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (coop) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// the same through an untyped kernel entry and an argument pointer array
inline cudaError_t launch_ex_c(const void* kernel, int grid, int threads, cudaStream_t stream, bool coop,
                               void** params) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (coop) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, kernel, params);
}

}  // namespace
