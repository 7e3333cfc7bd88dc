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

#include <cstdint>
#include <cstdlib>

using ss_internal::fail;

namespace {

constexpr int kMaxRanks = SS_SYMM_MAX_RANKS;
constexpr int kThreads = 512;

struct SymmArgs {
    float* bufs[kMaxRanks];      // peer buffer bases, index = rank
    uint64_t* pads[kMaxRanks];   // peer signal regions: [0, W) flag slots, [W, 2W) done slots
    float* mc;                   // multicast address of the buffer, nullptr -> P2P path
    int rank, world;
    int64_t n;
    int32_t* word;               // exchange: own word in, agreed word out; else: agreed word
    int exchange;
    float scale;
    uint32_t* seq;               // step counter (advanced by the last block)
    unsigned int* arrive;        // block arrival counter (self-resetting)
    int32_t* agreed_ring;        // optional: agreed word per step, ring of ring_cap
    int32_t ring_cap;
    int32_t* err;                // set to SS_SYMM_ERR_TIMEOUT on a timeout
    uint64_t timeout_ns;
};

__device__ __forceinline__ uint64_t now_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float4 mm_ld_reduce_add4(const float* p) {
    float4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ void mm_st4(float* p, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ float mm_ld_reduce_add1(const float* p) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void mm_st1(float* p, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// spin until (*p >> shift) == want (bounded); returns the last value read
__device__ uint64_t wait_tag(const uint64_t* p, uint64_t want, int shift, const SymmArgs& a, bool* timed_out) {
    const uint64_t t0 = now_ns();
    uint64_t v = ld_acquire_sys(p);
    while ((v >> shift) != want) {
        if (now_ns() - t0 > a.timeout_ns) {
            *timed_out = true;
            return v;
        }
        __nanosleep(64);
        v = ld_acquire_sys(p);
    }
    return v;
}

__device__ __forceinline__ float4 scale4(float4 v, float s) {
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    return v;
}

// Shard of rank r: vectors [v0, v1) of the n/4 float4s; the scalar tail goes to the last rank.
__device__ __forceinline__ void shard_range(const SymmArgs& a, int64_t* v0, int64_t* v1) {
    const int64_t nvec = a.n >> 2;
    const int64_t per = (nvec + a.world - 1) / a.world;
    *v0 = per * a.rank < nvec ? per * a.rank : nvec;
    *v1 = *v0 + per < nvec ? *v0 + per : nvec;
}

// NVLS: the switch reduces, multimem.st broadcasts (W = 0) -- or P2P two-shot
// over W peers: all W loads of U vectors issued before any add (fixed rank
// order => every rank's copy of a shard is bit-identical).
template <int W>
__device__ void average_shard(const SymmArgs& a) {
    int64_t v0, v1;
    shard_range(a, &v0, &v1);
    const int64_t nvec = a.n >> 2;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t i = v0 + tid;
    if constexpr (W == 0) {
        constexpr int U = 4;
        for (; i + (U - 1) * stride < v1; i += U * stride) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = mm_ld_reduce_add4(a.mc + 4 * (i + u * stride));
#pragma unroll
            for (int u = 0; u < U; ++u) mm_st4(a.mc + 4 * (i + u * stride), scale4(v[u], a.scale));
        }
        for (; i < v1; i += stride) mm_st4(a.mc + 4 * i, scale4(mm_ld_reduce_add4(a.mc + 4 * i), a.scale));
        if (a.rank == a.world - 1) {
            for (int64_t j = 4 * nvec + tid; j < a.n; j += stride)
                mm_st1(a.mc + j, mm_ld_reduce_add1(a.mc + j) * a.scale);
        }
    } else {
        constexpr int U = W <= 2 ? 4 : (W <= 4 ? 2 : 1);
        const float4* src[W];
        float4* dst[W];
#pragma unroll
        for (int r = 0; r < W; ++r) {
            src[r] = reinterpret_cast<const float4*>(a.bufs[r]);
            dst[r] = reinterpret_cast<float4*>(a.bufs[r]);
        }
        for (; i + (U - 1) * stride < v1; i += U * stride) {
            float4 v[U][W];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int r = 0; r < W; ++r) v[u][r] = __ldcg(src[r] + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float4 acc = v[u][0];
#pragma unroll
                for (int r = 1; r < W; ++r) {
                    acc.x += v[u][r].x; acc.y += v[u][r].y; acc.z += v[u][r].z; acc.w += v[u][r].w;
                }
                acc = scale4(acc, a.scale);
#pragma unroll
                for (int r = 0; r < W; ++r) __stcg(dst[r] + i + u * stride, acc);
            }
        }
        for (; i < v1; i += stride) {
            float4 acc = __ldcg(src[0] + i);
#pragma unroll
            for (int r = 1; r < W; ++r) {
                float4 v = __ldcg(src[r] + i);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            acc = scale4(acc, a.scale);
#pragma unroll
            for (int r = 0; r < W; ++r) __stcg(dst[r] + i, acc);
        }
        if (a.rank == a.world - 1) {
            for (int64_t j = 4 * nvec + tid; j < a.n; j += stride) {
                float acc = __ldcg(a.bufs[0] + j);
#pragma unroll
                for (int r = 1; r < W; ++r) acc += __ldcg(a.bufs[r] + j);
                acc *= a.scale;
#pragma unroll
                for (int r = 0; r < W; ++r) __stcg(a.bufs[r] + j, acc);
            }
        }
    }
}

template <int W>
__global__ void __launch_bounds__(kThreads) symm_sync_kernel(SymmArgs a) {
    __shared__ int s_word;
    __shared__ bool s_timeout;
    const uint64_t seq = static_cast<uint64_t>(*reinterpret_cast<volatile uint32_t*>(a.seq)) + 1;
    uint64_t* my_pad = a.pads[a.rank];
    if (threadIdx.x == 0) {
        bool timed_out = false;
        int w;
        if (a.exchange) {
            if (blockIdx.x == 0) {
                const int own = *a.word;
                __threadfence_system();
                const uint64_t v = (seq << 32) | static_cast<uint32_t>(own);
                for (int j = 0; j < a.world; ++j) st_release_sys(a.pads[j] + a.rank, v);
            }
            w = 0;
            for (int j = 0; j < a.world && !timed_out; ++j) {
                const uint64_t v = wait_tag(my_pad + j, seq, 32, a, &timed_out);
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
        average_shard<W>(a);
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int prev = atomicAdd(a.arrive, 1u);
        if (prev == gridDim.x - 1) {  // last block of this rank
            if (a.exchange) *a.word = w;
            if (a.agreed_ring && a.ring_cap > 0) a.agreed_ring[(seq - 1) % a.ring_cap] = s_timeout ? -1 : w;
            if (sync) {
                for (int j = 0; j < a.world; ++j) st_release_sys(a.pads[j] + a.world + a.rank, seq);
                bool timed_out = false;
                for (int j = 0; j < a.world && !timed_out; ++j) wait_tag(my_pad + a.world + j, seq, 0, a, &timed_out);
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
    static int override_grid = -1;
    if (override_grid < 0) {
        const char* e = getenv("SS_SYMM_GRID");
        override_grid = e ? atoi(e) : 0;
    }
    if (override_grid > 0 && override_grid < grid) grid = override_grid;
    const int64_t per_rank_vec = ((a.n >> 2) + a.world - 1) / a.world;
    const int64_t want = (per_rank_vec + kThreads * 4 - 1) / (kThreads * 4);
    if (want < grid) grid = static_cast<int>(want < 1 ? 1 : want);
    symm_sync_kernel<W><<<grid, kThreads, 0, s>>>(a);
    return ss_internal::check_launch("ss_symm_sync_f32");
}

}  // namespace

extern "C" {

int ss_symm_signal_bytes(int32_t world, int64_t* bytes) {
    if (!bytes) return fail(SS_ERR_CONFIG, "null output");
    if (world < 1 || world > kMaxRanks) return fail(SS_ERR_CONFIG, "world size must be in [1, %d], got %d", kMaxRanks, world);
    *bytes = 2 * static_cast<int64_t>(world) * static_cast<int64_t>(sizeof(uint64_t));
    return SS_OK;
}

int ss_symm_sync_f32(float* const* bufs, uint64_t* const* pads, float* mc, int32_t rank, int32_t world,
                     int64_t n, int32_t* word, int32_t exchange, float scale, uint32_t* seq, void* ws,
                     int32_t* agreed_ring, int32_t ring_cap, int32_t* err, double timeout_s, void* stream) {
    if (world < 1 || world > kMaxRanks) return fail(SS_ERR_CONFIG, "world size must be in [1, %d], got %d", kMaxRanks, world);
    if (rank < 0 || rank >= world) return fail(SS_ERR_CONFIG, "rank %d out of range for world %d", rank, world);
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0");
    if (!bufs || !pads || !word || !seq || !ws || !err) return fail(SS_ERR_CONFIG, "null pointer argument");
    if (ring_cap < 0 || (agreed_ring && ring_cap == 0)) return fail(SS_ERR_CONFIG, "bad agreed ring capacity");
    if (!(timeout_s > 0.0)) return fail(SS_ERR_CONFIG, "timeout must be positive");
    SymmArgs a;
    for (int r = 0; r < kMaxRanks; ++r) {
        a.bufs[r] = nullptr;
        a.pads[r] = nullptr;
    }
    for (int r = 0; r < world; ++r) {
        if (!bufs[r] || !pads[r]) return fail(SS_ERR_CONFIG, "null peer pointer for rank %d", r);
        if ((reinterpret_cast<uintptr_t>(bufs[r]) & 15) != 0) return fail(SS_ERR_CONFIG, "peer buffer %d not 16-byte aligned", r);
        a.bufs[r] = bufs[r];
        a.pads[r] = pads[r];
    }
    if (mc && (reinterpret_cast<uintptr_t>(mc) & 15) != 0) return fail(SS_ERR_CONFIG, "multicast address not 16-byte aligned");
    a.mc = mc;
    a.rank = rank;
    a.world = world;
    a.n = n;
    a.word = word;
    a.exchange = exchange ? 1 : 0;
    a.scale = scale;
    a.seq = seq;
    a.arrive = static_cast<unsigned int*>(ws);
    a.agreed_ring = agreed_ring;
    a.ring_cap = ring_cap;
    a.err = err;
    a.timeout_ns = static_cast<uint64_t>(timeout_s * 1e9);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (mc) return launch_symm<0>(a, s);
    switch (world) {
        case 1: return launch_symm<1>(a, s);
        case 2: return launch_symm<2>(a, s);
        case 3: return launch_symm<3>(a, s);
        case 4: return launch_symm<4>(a, s);
        case 5: return launch_symm<5>(a, s);
        case 6: return launch_symm<6>(a, s);
        case 7: return launch_symm<7>(a, s);
        case 8: return launch_symm<8>(a, s);
        default:
            return fail(SS_ERR_CONFIG, "the P2P path supports up to 8 ranks; use multicast for %d", world);
    }
}

}  // extern "C"
