// selsync_step.cu -- the whole SelSync step from ONE host launch.
//
// Reference path (/root/reference/pkg/src/selsync): _selsync_step
// (strategies.py:369-403) with the parameter server's flag relay
// (runtime.py:319-333) and mean round (runtime.py:275-294). On the device:
// update + ||g||^2 + signal (K13+K2) -> vote exchange over NVLink (C1) ->
// on sync only, a dynamically launched NVLink mean (C2).

#include "selsync_b200.h"
#include "common.cuh"
#include "device_core.cuh"
#include "host_util.cuh"
#include "symm_device.cuh"

#include <cuda_runtime.h>

#include <cstdint>

using ss_internal::check_launch;
using ss_internal::fail;

namespace {

// ------------------------------------------- the whole step in one host launch
//
// step_kernel: K13 (update + ||g||^2) over the whole buffer; the last block
// to arrive reduces the partials, runs K2, posts its vote to every peer's
// signal slot and waits for the N votes (C1: MAX = OR). Every other block has
// already exited, so a local step costs the update plus one NVLink round trip
// in a single block. On sync the last block tail-launches avg_kernel (CUDA
// dynamic parallelism, cudaStreamTailLaunch: it starts once this grid has
// fully retired) which averages this rank's shard over NVLink with the 1/N in
// the epilogue (C2) and closes with the end barrier. One host launch per step,
// the branch never leaves the device.
template <int W>
__global__ void __launch_bounds__(512, 2) avg_kernel(SymmArgs s, uint64_t seq) {
    average_shard<W>(s);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(s.arrive, 1u) == gridDim.x - 1) {
        for (int j = 0; j < s.world; ++j) st_release_sys(s.pads[j] + s.world + s.rank, seq);
        bool to = false;
        for (int j = 0; j < s.world && !to; ++j) wait_tag(s.pads[s.rank] + s.world + j, seq, 0, s, &to);
        if (to) atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
        *s.arrive = 0u;
        *s.seq = static_cast<uint32_t>(seq);
    }
}

template <bool MOM, bool NEST, int W>
__global__ void __launch_bounds__(kThreads, 4) step_kernel(SgdArgs a, Finish f, SymmArgs s, int avg_grid) {
    __shared__ bool s_last;
    const double acc = sgd_pass<MOM, NEST, true, (MOM ? 1 : 2)>(a);
    Workspace ws = ws_view(f.ws);
    const double bsum = block_sum(acc);
    if (threadIdx.x == 0) {
        ws.partials[blockIdx.x] = bsum;
        __threadfence_system();  // this block's parameter stores reach peers before the vote
        s_last = atomicAdd(ws.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double v = 0.0;
    for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += blockDim.x) v += __ldcg(ws.partials + i);
    v = block_sum(v);
    if (threadIdx.x != 0) return;
    *ws.counter = 0u;
    const uint64_t seq = static_cast<uint64_t>(*reinterpret_cast<volatile uint32_t*>(s.seq)) + 1;
    signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
    const uint64_t tagged = (seq << 32) | static_cast<uint32_t>(*f.word);
    __threadfence_system();
    for (int j = 0; j < s.world; ++j) st_release_sys(s.pads[j] + s.rank, tagged);
    bool to = false;
    int w = 0;
    for (int j = 0; j < s.world && !to; ++j) {
        const uint64_t t = wait_tag(s.pads[s.rank] + j, seq, 32, s, &to);
        const int wj = static_cast<int>(static_cast<uint32_t>(t));
        w = wj > w ? wj : w;
    }
    if (to) {
        atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
        w = -1;
    }
    *f.word = w;
    if (s.agreed_ring && s.ring_cap > 0) s.agreed_ring[(seq - 1) % s.ring_cap] = w;
    if (w == SS_FLAG_SYNC) {
        avg_kernel<W><<<avg_grid, 512, 0, cudaStreamTailLaunch>>>(s, seq);
    } else {
        *s.seq = static_cast<uint32_t>(seq);
    }
}

}  // namespace

namespace {

template <bool MOM, bool NEST, int W>
int launch_step(const SgdArgs& a, Finish f, const SymmArgs& sa, void* stream) {
    static int resident = 0, avg_resident = 0;
    if (resident == 0) {
        int x = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, step_kernel<MOM, NEST, W>, kThreads, 0) != cudaSuccess || x <= 0)
            x = 1;
        resident = x;
        x = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, avg_kernel<W>, 512, 0) != cudaSuccess || x <= 0) x = 1;
        avg_resident = x;
    }
    const int grid = static_cast<int>(grid_for((a.n - a.head) / 4 + 1, MOM ? 1 : 2, resident));
    f.total_blocks = grid;
    // averaging grid: every block co-resident (the last one runs the end barrier)
    int avg_grid = ss_internal::sm_count() * avg_resident;
    const int64_t per_rank_vec = ((sa.n >> 2) + sa.world - 1) / sa.world;
    const int64_t want = (per_rank_vec + 512 * 4 - 1) / (512 * 4);
    if (want < avg_grid) avg_grid = static_cast<int>(want < 1 ? 1 : want);
    step_kernel<MOM, NEST, W><<<grid, kThreads, 0, as_stream(stream)>>>(a, f, sa, avg_grid);
    return check_launch("ss_step_symm_f32");
}

template <int W>
int dispatch_step(const SgdArgs& a, const Finish& f, const SymmArgs& sa, bool mom, bool nest, void* stream) {
    if (!mom) return launch_step<false, false, W>(a, f, sa, stream);
    if (nest) return launch_step<true, true, W>(a, f, sa, stream);
    return launch_step<true, false, W>(a, f, sa, stream);
}

}  // namespace

extern "C" int ss_step_symm_f32(float* w, const float* g, float* m, int64_t n, float lr, float momentum,
                                float dampening, float weight_decay, int32_t nesterov, int32_t first_step,
                                ss_signal_state* st, double delta, int32_t* word, ss_trace_row* trace,
                                int32_t cap, const ss_symm_group* grp, void* ws, void* stream) {
    SgdArgs a;
    int rc = make_sgd_args(&a, w, g, m, n, lr, momentum, dampening, weight_decay, nesterov, first_step,
                           nullptr, 1.0f);
    if (rc) return rc;
    if (!st || !ws || !word) return fail(SS_ERR_CONFIG, "null state/word/workspace");
    rc = check_delta_impl(delta);
    if (rc) return rc;
    rc = check_trace(trace, cap);
    if (rc) return rc;
    SymmArgs sa;
    rc = symm_args_from_group(grp, n, word, 1, 1.0f / static_cast<float>(grp ? grp->world : 1), ws, &sa,
                              &ss_internal::fail);
    if (rc) return rc;
    if (grp->bufs[grp->rank] != w) return fail(SS_ERR_CONFIG, "w must be this rank's symmetric buffer");
    Finish f{ws, 0, 0, nullptr, st, delta, word, trace, cap};
    const bool mom = momentum != 0.0f, nest = nesterov != 0;
    switch (symm_width(sa)) {
        case 0: return dispatch_step<0>(a, f, sa, mom, nest, stream);
        case 2: return dispatch_step<2>(a, f, sa, mom, nest, stream);
        case 4: return dispatch_step<4>(a, f, sa, mom, nest, stream);
        case 8: return dispatch_step<8>(a, f, sa, mom, nest, stream);
        default:
            return fail(SS_ERR_CONFIG, "one-launch step: world %d needs multicast (P2P widths 2, 4, 8)", sa.world);
    }
}
