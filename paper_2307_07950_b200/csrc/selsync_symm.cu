// selsync_symm.cu -- device-side SelSync exchange over NVLink peer memory.
//
// Replaces the parameter server's two reactions of a SelSync step
// (reference /root/reference/pkg/src/selsync):
//   flag relay   runtime.py:319-333 (+ wire.py:139-151)  -> optional P2P flag exchange (C1)
//   mean round   runtime.py:275-294 -> strategies.py:159-168 -> conditional averaging (C2)
// with ONE kernel that reads the agreed flag word on the device, so no rank
// ever needs the host to learn the branch (no host round-trip, CUDA-graph
// capturable). The flat fp32 parameter buffer lives in symmetric memory
// (torch.distributed._symmetric_memory): every rank holds the peer addresses
// of all N buffers and, when the NVSwitch supports it, one multicast address.
//
// Sync step, multicast (NVLS) path: rank r owns shard r of the buffer;
//   multimem.ld_reduce.add.v4.f32 pulls the N-way sum of a 16-byte vector
//   through the switch, the 1/N scale is applied in registers (the epilogue),
//   multimem.st.v4.f32 broadcasts the mean into every rank's buffer.
// P2P path (no multicast): rank r reads shard r from every peer in rank order
// (fixed summation order), scales, and stores the mean to every peer.
//
// Ordering: C1 (NCCL allreduce-MAX, or the P2P exchange here) completes only
// after every rank's update kernel finished, so all buffers are final before
// anyone reads; an end barrier keeps every rank from starting its next update
// while a peer still reads or writes its buffer. Every spin is bounded by a
// timeout that sets an error word instead of hanging the GPU.

#include "selsync_b200.h"
#include "common.cuh"

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>

using ss_internal::fail;

#include "symm_device.cuh"

namespace {

// block shape of the standalone exchange (A/B builds: SS_SYMM_THREADS / SS_SYMM_MINB)
#ifndef SS_SYMM_THREADS
#define SS_SYMM_THREADS 512
#endif
#ifndef SS_SYMM_MINB
#define SS_SYMM_MINB 2
#endif
constexpr int kThreads = SS_SYMM_THREADS;

template <int W>
__global__ void __launch_bounds__(kThreads, SS_SYMM_MINB) symm_sync_kernel(SymmArgs a) {
    __shared__ int s_word;
    __shared__ bool s_timeout;
    const uint64_t seq = static_cast<uint64_t>(*reinterpret_cast<volatile uint32_t*>(a.seq)) + 1;
    if (threadIdx.x == 0) {
        bool timed_out = false;
        int w;
        if (a.exchange) {
            if (blockIdx.x == 0) {
                const int own = *a.word;
                const uint64_t v = (seq << 32) | static_cast<uint32_t>(own);
                fence_acq_rel_sys();
                for (int j = 0; j < a.world; ++j) st_relaxed_sys(vote_slot(a, j, seq, a.rank), v);
            }
            w = 0;
            for (int j = 0; j < a.world && !timed_out; ++j) {
                const uint64_t v = wait_tag(vote_slot(a, a.rank, seq, j), seq, 32, a, &timed_out);
                const int wj = static_cast<int>(static_cast<uint32_t>(v));
                w = wj > w ? wj : w;
            }
        } else {
            w = *a.word;
        }
        s_word = w;
        s_timeout = timed_out;
        if (timed_out) atomicExch(a.err, SS_SYMM_ERR_TIMEOUT);
    }
    __syncthreads();
    const int w = s_word;
    const bool sync = !s_timeout && w == SS_FLAG_SYNC;
    if (sync) {
        average_shard<W>(a, hw_blk());
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(a.arrive, 1u);
        if (prev == gridDim.x - 1) {  // last block of this rank
            if (a.exchange) *a.word = w;
            if (a.agreed_ring && a.ring_cap > 0) a.agreed_ring[(seq - 1) % a.ring_cap] = s_timeout ? -1 : w;
            if (sync) {
                fence_acq_rel_sys();
                for (int j = 0; j < a.world; ++j) st_relaxed_sys(done_slot(a, j, a.rank), seq);
                bool timed_out = false;
                for (int j = 0; j < a.world && !timed_out; ++j) wait_tag(done_slot(a, a.rank, j), seq, 0, a, &timed_out);
                if (timed_out) atomicExch(a.err, SS_SYMM_ERR_TIMEOUT);
            }
            *a.arrive = 0u;
            *a.seq = static_cast<uint32_t>(seq);
        }
    }
}

template <int W>
int launch_symm(const SymmArgs& a, cudaStream_t s) {
    static int resident = 0;
    if (resident == 0) {
        int x = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, symm_sync_kernel<W>, kThreads, 0) != cudaSuccess || x <= 0) x = 1;
        resident = x;
    }
    // all blocks co-resident: they never wait on each other, but the last
    // block's end barrier must not be starved behind queued blocks
    int grid = ss_internal::sm_count() * resident;
    const int64_t per_rank_vec = ((a.n >> 2) + a.world - 1) / a.world;
    const int64_t want = (per_rank_vec + kThreads * 4 - 1) / (kThreads * 4);
    if (want < grid) grid = static_cast<int>(want < 1 ? 1 : want);
    symm_sync_kernel<W><<<grid, kThreads, 0, s>>>(a);
    return ss_internal::check_launch("ss_symm_sync_f32");
}

}  // namespace

extern "C" {

int ss_symm_group_layout(int64_t* offsets, int32_t cap, int32_t* count) {
    const int64_t o[] = {
        (int64_t)offsetof(ss_symm_group, bufs),        (int64_t)offsetof(ss_symm_group, pads),
        (int64_t)offsetof(ss_symm_group, mc),          (int64_t)offsetof(ss_symm_group, seq),
        (int64_t)offsetof(ss_symm_group, agreed_ring), (int64_t)offsetof(ss_symm_group, err),
        (int64_t)offsetof(ss_symm_group, timeout_s),   (int64_t)offsetof(ss_symm_group, rank),
        (int64_t)offsetof(ss_symm_group, world),       (int64_t)offsetof(ss_symm_group, ring_cap),
        (int64_t)offsetof(ss_symm_group, max_blocks),    (int64_t)offsetof(ss_symm_group, order_mode),
        (int64_t)offsetof(ss_symm_group, order_threshold), (int64_t)offsetof(ss_symm_group, tile_cnt),
        (int64_t)offsetof(ss_symm_group, epoch),       (int64_t)offsetof(ss_symm_group, predictor),
        (int64_t)offsetof(ss_symm_group, tile_elems),  (int64_t)offsetof(ss_symm_group, n_tiles),
        (int64_t)offsetof(ss_symm_group, tile_norm),   (int64_t)offsetof(ss_symm_group, debug_events),
        (int64_t)offsetof(ss_symm_group, debug_cap),   (int64_t)sizeof(ss_symm_group)};
    const int32_t n = static_cast<int32_t>(sizeof(o) / sizeof(o[0]));
    if (!offsets || !count) return fail(SS_ERR_CONFIG, "null argument");
    if (cap < n) return fail(SS_ERR_CONFIG, "layout needs %d entries, got room for %d", n, cap);
    for (int32_t i = 0; i < n; ++i) offsets[i] = o[i];
    *count = n;
    return SS_OK;
}

int ss_rank_step_layout(int64_t* offsets, int32_t cap, int32_t* count) {
    const int64_t o[] = {
        (int64_t)offsetof(ss_rank_step, w_dev),        (int64_t)offsetof(ss_rank_step, g_dev),
        (int64_t)offsetof(ss_rank_step, m_dev),        (int64_t)offsetof(ss_rank_step, n),
        (int64_t)offsetof(ss_rank_step, momentum),     (int64_t)offsetof(ss_rank_step, dampening),
        (int64_t)offsetof(ss_rank_step, weight_decay), (int64_t)offsetof(ss_rank_step, nesterov),
        (int64_t)offsetof(ss_rank_step, st_dev),       (int64_t)offsetof(ss_rank_step, delta),
        (int64_t)offsetof(ss_rank_step, word_dev),     (int64_t)offsetof(ss_rank_step, trace_dev),
        (int64_t)offsetof(ss_rank_step, trace_cap),    (int64_t)offsetof(ss_rank_step, reserved),
        (int64_t)offsetof(ss_rank_step, group),        (int64_t)offsetof(ss_rank_step, ws_dev),
        (int64_t)sizeof(ss_rank_step),                 (int64_t)sizeof(ss_step_plan)};
    const int32_t n = static_cast<int32_t>(sizeof(o) / sizeof(o[0]));
    if (!offsets || !count) return fail(SS_ERR_CONFIG, "null argument");
    if (cap < n) return fail(SS_ERR_CONFIG, "layout needs %d entries, got room for %d", n, cap);
    for (int32_t i = 0; i < n; ++i) offsets[i] = o[i];
    *count = n;
    return SS_OK;
}

int ss_symm_signal_bytes(int32_t world, int64_t* bytes) {
    if (!bytes) return fail(SS_ERR_CONFIG, "null output");
    if (world < 1 || world > kMaxRanks) return fail(SS_ERR_CONFIG, "world size must be in [1, %d], got %d", kMaxRanks, world);
    *bytes = 5 * static_cast<int64_t>(world) * static_cast<int64_t>(sizeof(uint64_t));
    return SS_OK;
}

int ss_symm_sync_f32(const ss_symm_group* g, int64_t n, int32_t* word, int32_t exchange, float scale,
                     void* ws, void* stream) {
    SymmArgs a;
    int rc = symm_args_from_group(g, n, word, exchange, scale, ws, &a, &ss_internal::fail);
    if (rc) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (symm_width(a)) {
        case 0: return launch_symm<0>(a, s);
        case 1: return launch_symm<1>(a, s);
        case 2: return launch_symm<2>(a, s);
        case 3: return launch_symm<3>(a, s);
        case 4: return launch_symm<4>(a, s);
        case 5: return launch_symm<5>(a, s);
        case 6: return launch_symm<6>(a, s);
        case 7: return launch_symm<7>(a, s);
        case 8: return launch_symm<8>(a, s);
        default:
            return fail(SS_ERR_CONFIG, "the P2P path supports up to 8 ranks; use multicast for %d", a.world);
    }
}

}  // extern "C"
