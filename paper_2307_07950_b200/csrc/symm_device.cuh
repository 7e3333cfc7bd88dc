// symm_device.cuh -- device helpers for the NVLink peer-memory exchange,
// shared by the standalone exchange kernel (selsync_symm.cu) and the fused
// one-launch step kernel (selsync_b200.cu). Internal; not part of the C-ABI.
#pragma once

#include "selsync_b200.h"
#include "common.cuh"

#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kMaxRanks = SS_SYMM_MAX_RANKS;
struct SymmArgs {
    float* bufs[kMaxRanks];      // peer buffer bases, index = rank
    uint64_t* pads[kMaxRanks];   // peer signal regions: 2 x W vote slots (by seq parity), W done slots
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

// A release pattern to several peers: ONE fence, then relaxed system-scope
// stores (PTX: a strong write preceded by fence.acq_rel is a release). N
// st.release.sys in a row would each wait for the previous remote store to be
// acknowledged over NVLink before issuing the next.
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// NVLS tuning (A/B builds, tools/ab_build.sh): SS_NVLS_WEAK=1 uses .weak
// instead of .relaxed.sys; SS_NVLS_U sets the 16-byte vectors per thread in flight
#ifndef SS_NVLS_WEAK
#define SS_NVLS_WEAK 0
#endif
#ifndef SS_NVLS_U
#define SS_NVLS_U 4
#endif
// 16-byte vectors in flight per thread in the per-tile means of the
// overlapped sync step (one block per tile): NVLS reductions, P2P vectors per rank
#ifndef SS_TILE_U_NVLS
#define SS_TILE_U_NVLS 2
#endif
#ifndef SS_TILE_U_P2P
#define SS_TILE_U_P2P 2
#endif

__device__ __forceinline__ float4 mm_ld_reduce_add4(const float* p) {
    float4 v;
#if SS_NVLS_WEAK
    asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
#else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
#endif
    return v;
}

__device__ __forceinline__ void mm_st4(float* p, float4 v) {
#if SS_NVLS_WEAK
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
#else
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
#endif
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

__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// spin (bounded) until a gpu-scope tag (*p >> 32) == want; returns the last
// value. Up to a few hundred blocks poll one word while the slowest blocks
// still stream: relaxed polls with a back-off keep that traffic light, one
// acquire fence after the match orders what follows.
__device__ uint64_t wait_tag_gpu(const uint64_t* p, uint64_t want, uint64_t timeout_ns, bool* timed_out,
                                 unsigned sleep_ns = 256) {
    const uint64_t t0 = now_ns();
    uint64_t v = ld_relaxed_gpu(p);
    while ((v >> 32) != want) {
        if (now_ns() - t0 > timeout_ns) {
            *timed_out = true;
            return v;
        }
        __nanosleep(sleep_ns);
        v = ld_relaxed_gpu(p);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return v;
}

// Signal slots of rank `owner`'s region. Votes are double-buffered by the
// parity of the step tag: a fast rank may post its vote for step s+1 before a
// slow rank has read the step-s votes, but never for s+2 (that needs the slow
// rank's s+1 vote, posted only after it read all step-s votes).
__device__ __forceinline__ uint64_t* vote_slot(const SymmArgs& a, int owner, uint64_t seq, int from) {
    return a.pads[owner] + (seq & 1) * a.world + from;
}
__device__ __forceinline__ uint64_t* done_slot(const SymmArgs& a, int owner, int from) {
    return a.pads[owner] + 2 * a.world + from;
}
// poison tags (seq of the step): rank `from` met a NaN gradient in an update
// tile of the known-sync pass, whose mean runs before the vote is in
__device__ __forceinline__ uint64_t* poison_slot(const SymmArgs& a, int owner, int from) {
    return a.pads[owner] + 3 * a.world + from;
}
// early sync tags (seq of the step): rank `from`'s running lower bound of
// ||g||^2 proved its vote sync before its sweep ended (exact early vote)
__device__ __forceinline__ uint64_t* early_slot(const SymmArgs& a, int owner, int from) {
    return a.pads[owner] + 4 * a.world + from;
}

// peer load / store flavours of the P2P mean (tuning: SS_P2P_VARIANT)
template <int LS>
__device__ __forceinline__ float4 p2p_ld(const float4* p) {
    if constexpr (LS == 1) return *p;
    else if constexpr (LS == 3) return __ldcs(p);
    else return __ldcg(p);
}
template <int LS>
__device__ __forceinline__ void p2p_st(float4* p, float4 v) {
    if constexpr (LS == 1) *p = v;
    else if constexpr (LS == 2 || LS == 3) __stcs(p, v);
    else __stcg(p, v);
}

__device__ __forceinline__ float4 scale4(float4 v, float s) {
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    return v;
}

// Mean over ranks of elements [e0, e1) by the threads of ONE block (tile work
// of the overlapped sync step); e0 % 4 == 0, scalar tail when e1 % 4 != 0.
template <int W>
__device__ void average_block_range(const SymmArgs& a_in, int64_t e0, int64_t e1) {
    // register copy of what the loops use (a_in may live in shared memory)
    SymmArgs a;
    a.mc = a_in.mc;
    a.scale = a_in.scale;
#pragma unroll
    for (int r = 0; r < (W > 0 ? W : 1); ++r) a.bufs[r] = a_in.bufs[r];
    const int64_t v0 = e0 >> 2, v1 = e1 >> 2;
    if constexpr (W == 0) {
        constexpr int U = SS_TILE_U_NVLS;  // multimem reductions in flight per thread
        const int64_t bs = blockDim.x;
        int64_t i = v0 + threadIdx.x;
        for (; i + (U - 1) * bs < v1; i += U * bs) {
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = mm_ld_reduce_add4(a.mc + 4 * (i + u * bs));
#pragma unroll
            for (int u = 0; u < U; ++u) mm_st4(a.mc + 4 * (i + u * bs), scale4(x[u], a.scale));
        }
        for (; i < v1; i += bs) mm_st4(a.mc + 4 * i, scale4(mm_ld_reduce_add4(a.mc + 4 * i), a.scale));
        for (int64_t j = 4 * v1 + threadIdx.x; j < e1; j += blockDim.x)
            mm_st1(a.mc + j, mm_ld_reduce_add1(a.mc + j) * a.scale);
    } else {
        constexpr int U = W <= 2 ? SS_TILE_U_P2P : (W <= 4 ? 2 : 1);  // peer loads in flight per thread: U * W
        const int64_t bs = blockDim.x;
        int64_t i = v0 + threadIdx.x;
        for (; i + (U - 1) * bs < v1; i += U * bs) {
            float4 v[U][W];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int r = 0; r < W; ++r) v[u][r] = __ldcg(reinterpret_cast<const float4*>(a.bufs[r]) + i + u * bs);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float4 acc = v[u][0];
#pragma unroll
                for (int r = 1; r < W; ++r) {
                    acc.x += v[u][r].x; acc.y += v[u][r].y; acc.z += v[u][r].z; acc.w += v[u][r].w;
                }
                acc = scale4(acc, a.scale);
#pragma unroll
                for (int r = 0; r < W; ++r) __stcg(reinterpret_cast<float4*>(a.bufs[r]) + i + u * bs, acc);
            }
        }
        for (; i < v1; i += bs) {
            float4 v[W];
#pragma unroll
            for (int r = 0; r < W; ++r) v[r] = __ldcg(reinterpret_cast<const float4*>(a.bufs[r]) + i);
            float4 acc = v[0];
#pragma unroll
            for (int r = 1; r < W; ++r) {
                acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w;
            }
            acc = scale4(acc, a.scale);
#pragma unroll
            for (int r = 0; r < W; ++r) __stcg(reinterpret_cast<float4*>(a.bufs[r]) + i, acc);
        }
        for (int64_t j = 4 * v1 + threadIdx.x; j < e1; j += bs) {
            float acc = __ldcg(a.bufs[0] + j);
#pragma unroll
            for (int r = 1; r < W; ++r) acc += __ldcg(a.bufs[r] + j);
            acc *= a.scale;
#pragma unroll
            for (int r = 0; r < W; ++r) __stcg(a.bufs[r] + j, acc);
        }
    }
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
template <int W, int UO = 0, int LS = 0>
__device__ void average_shard(const SymmArgs& a_in, VBlk vb) {
    SymmArgs a;  // register copy of what the loops use (a_in may live in shared memory)
    a.mc = a_in.mc;
    a.scale = a_in.scale;
    a.n = a_in.n;
    a.rank = a_in.rank;
    a.world = a_in.world;
#pragma unroll
    for (int r = 0; r < (W > 0 ? W : 1); ++r) a.bufs[r] = a_in.bufs[r];
    int64_t v0, v1;
    shard_range(a, &v0, &v1);
    const int64_t nvec = a.n >> 2;
    const int64_t tid = static_cast<int64_t>(vb.bid) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(vb.n) * blockDim.x;
    int64_t i = v0 + tid;
    if constexpr (W == 0) {
        constexpr int U = UO ? UO : SS_NVLS_U;
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
        constexpr int U = UO ? UO : (W <= 2 ? 4 : (W <= 4 ? 2 : 1));
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
                for (int r = 0; r < W; ++r) v[u][r] = p2p_ld<LS>(src[r] + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float4 acc = v[u][0];
#pragma unroll
                for (int r = 1; r < W; ++r) {
                    acc.x += v[u][r].x; acc.y += v[u][r].y; acc.z += v[u][r].z; acc.w += v[u][r].w;
                }
                acc = scale4(acc, a.scale);
#pragma unroll
                for (int r = 0; r < W; ++r) p2p_st<LS>(dst[r] + i + u * stride, acc);
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


}  // namespace

namespace {

// Validate a host ss_symm_group and build the kernel argument block.
// ws: a zeroed ss_workspace; the exchange kernels use the arrival counter at
// byte 64 (the norm reductions own the one at byte 0).
inline int symm_args_from_group(const ss_symm_group* g, int64_t n, int32_t* word, int exchange,
                                float scale, void* ws, SymmArgs* a, int (*fail_fn)(int, const char*, ...)) {
    if (!g || !word || !ws) return fail_fn(SS_ERR_CONFIG, "null pointer argument");
    if (g->world < 1 || g->world > kMaxRanks)
        return fail_fn(SS_ERR_CONFIG, "world size must be in [1, %d], got %d", kMaxRanks, g->world);
    if (g->rank < 0 || g->rank >= g->world)
        return fail_fn(SS_ERR_CONFIG, "rank %d out of range for world %d", g->rank, g->world);
    if (n < 0) return fail_fn(SS_ERR_CONFIG, "n must be >= 0");
    if (!g->seq || !g->err) return fail_fn(SS_ERR_CONFIG, "null seq/err pointer in the group");
    if (g->ring_cap < 0 || (g->agreed_ring && g->ring_cap == 0))
        return fail_fn(SS_ERR_CONFIG, "bad agreed ring capacity");
    if (!(g->timeout_s > 0.0)) return fail_fn(SS_ERR_CONFIG, "timeout must be positive");
    for (int r = 0; r < kMaxRanks; ++r) {
        a->bufs[r] = nullptr;
        a->pads[r] = nullptr;
    }
    for (int r = 0; r < g->world; ++r) {
        if (!g->bufs[r] || !g->pads[r]) return fail_fn(SS_ERR_CONFIG, "null peer pointer for rank %d", r);
        if ((reinterpret_cast<uintptr_t>(g->bufs[r]) & 15) != 0)
            return fail_fn(SS_ERR_CONFIG, "peer buffer %d not 16-byte aligned", r);
        a->bufs[r] = g->bufs[r];
        a->pads[r] = g->pads[r];
    }
    if (g->mc && (reinterpret_cast<uintptr_t>(g->mc) & 15) != 0)
        return fail_fn(SS_ERR_CONFIG, "multicast address not 16-byte aligned");
    a->mc = g->mc;
    a->rank = g->rank;
    a->world = g->world;
    a->n = n;
    a->word = word;
    a->exchange = exchange ? 1 : 0;
    a->scale = scale;
    a->seq = g->seq;
    a->arrive = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + 64);
    a->agreed_ring = g->agreed_ring;
    a->ring_cap = g->ring_cap;
    a->err = g->err;
    a->timeout_ns = static_cast<uint64_t>(g->timeout_s * 1e9);
    return SS_OK;
}

// P2P template width for a world size (0 = NVLS multicast path); -1 = unsupported
inline int symm_width(const SymmArgs& a) {
    if (a.mc) return 0;
    return a.world <= 8 ? a.world : -1;
}

}  // namespace
