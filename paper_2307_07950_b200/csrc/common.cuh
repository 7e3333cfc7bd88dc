// common.cuh -- internal helpers shared by the translation units of
// libselsync_b200.so (not part of the C-ABI; hidden visibility).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ss_internal {

// record an error message for ss_last_error() and return `code`
int fail(int code, const char* fmt, ...);
// SS_OK or SS_ERR_CUDA with the pending launch error
int check_launch(const char* what);
// multiprocessor count of the current device
int sm_count();

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

}  // namespace
