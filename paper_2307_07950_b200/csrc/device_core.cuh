// device_core.cuh -- device code shared by the translation units of
// libselsync_b200.so: constants, workspace layout, the exact-IEEE signal step
// (K2), streaming memory helpers, block reductions with the deterministic
// two-pass finish, and the SGD element/pass templates (K3 / K13).
// Internal; not part of the C-ABI.
#pragma once

#include "selsync_b200.h"
#include "common.cuh"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <limits>

namespace {

// ---------------------------------------------------------------- constants

constexpr int kThreads = 256;
constexpr int kMaxGrid = 8192;
constexpr int64_t kWsHeader = 256;  // arrival counter, padded to its own sector group
constexpr int kMtMax = 256;         // tensors per multi-tensor launch (kernel-param table)
constexpr int kMaxReplicas = 64;
constexpr int kNormUnroll = 4;

struct Workspace {
    unsigned int* counter;
    double* partials;
};

__host__ __device__ inline Workspace ws_view(void* ws) {
    char* b = static_cast<char*>(ws);
    return Workspace{reinterpret_cast<unsigned int*>(b), reinterpret_cast<double*>(b + kWsHeader)};
}
// header: norm arrival counter at 0, exchange arrival counter at 64, ticket at
// 128, the early vote's running sum at 160 and posted tag at 176, the
// update-first step's decision broadcast at 192, the one-launch step's
// block-start counter at 224; then the partials
constexpr int64_t kWsBytes = kWsHeader + 8 * kMaxGrid;

// ------------------------------------------- exact IEEE scalar arithmetic
// The signal math must round exactly like the reference's Python floats:
// one rounding per operation, no FMA contraction (host side is compiled with
// -ffp-contract=off, device side uses the _rn intrinsics).

__host__ __device__ inline double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ inline double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ inline double sub_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
__host__ __device__ inline double div_rn(double a, double b) {
#ifdef __CUDA_ARCH__
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}
__host__ __device__ inline double d_inf() {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(0x7ff0000000000000LL);
#else
    return std::numeric_limits<double>::infinity();
#endif
}
__host__ __device__ inline double d_nan() {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(0x7ff8000000000000LL);
#else
    return std::numeric_limits<double>::quiet_NaN();
#endif
}

// relative_change, signal.py:86-98 (step_count >= 2 checked by callers)
__host__ __device__ inline double rel_change_core(double prev, double cur) {
    if (prev == 0.0) return cur == 0.0 ? 0.0 : d_inf();
    return fabs(div_rn(sub_rn(cur, prev), prev));
}

// observe, signal.py:64-83. Returns SS_FLAG_ERR_* bits; *s untouched on error.
__host__ __device__ inline int observe_core(ss_signal_state* s, double x) {
    if (x != x) return SS_FLAG_ERR_NAN;
    if (x < 0.0) return SS_FLAG_ERR_NEG;
    double cur;
    if (s->step_count == 0) {
        cur = x;  // seed the series at the first observation
    } else {
        cur = add_rn(mul_rn(s->smoothing, x), mul_rn(sub_rn(1.0, s->smoothing), s->ewma_current));
    }
    s->ewma_previous = s->ewma_current;
    s->ewma_current = cur;
    s->step_count += 1;
    s->last_norm_sq = x;
    if (s->step_count >= 2) {
        double d = rel_change_core(s->ewma_previous, s->ewma_current);
        s->last_delta = d;
        // Python max(a, b) keeps a unless b > a (NaN never wins)
        if (s->step_count > s->warmup && d > s->max_delta_seen) s->max_delta_seen = d;
    } else {
        s->last_delta = d_nan();
    }
    return 0;
}

// decide, signal.py:101-107, for step_count >= 1: warmup syncs, inclusive test
__host__ __device__ inline int vote_core(const ss_signal_state* s, double delta) {
    if (s->step_count <= s->warmup) return 1;
    return rel_change_core(s->ewma_previous, s->ewma_current) >= delta ? 1 : 0;
}

// The decision after the NEXT observation is sync whatever the observed norm
// (>= 0, not NaN): the observation about to be made is number <= warmup, or
// delta == 0 with a finite ewma_current (then Delta >= 0, inf included; an
// infinite EWMA would give Delta = inf/inf = NaN, i.e. "local"). Sound and
// complete: otherwise observing x == ewma_current gives Delta == 0 < delta,
// or NaN (local). tests/test_signal_api.py checks both directions.
__host__ __device__ inline bool sync_known_ahead_core(int64_t step_count, int32_t warmup, double delta,
                                                      double ewma_current) {
    if (step_count + 1 <= static_cast<int64_t>(warmup)) return true;
    return delta == 0.0 && ewma_current - ewma_current == 0.0;  // finite
}

// Exact early vote: `lower` is a partial sum of the non-negative terms whose
// total the finishing block will observe (the same block partials, a subset,
// summed in another order). If observing a value a little below `lower`
// already votes sync on the upward side (new EWMA >= previous), then so does
// the total: every operation of observe / relative_change rounds monotonically
// in x there, and the margin (1e-9 relative) covers the two summation orders
// (their difference is < 1e-12 relative for <= 8192 partials). Downward
// jumps are never proven early (they need an upper bound). NaN / inf-times-0
// give false. tests/test_signal_api.py checks soundness against the scalar
// vote of every total >= lower.
__host__ __device__ inline bool sync_proven_early_core(const ss_signal_state* st, double lower, double delta) {
    if (!(lower >= 0.0) || st->step_count < 1 || !(st->smoothing > 0.0)) return false;
    ss_signal_state s = *st;
    if (observe_core(&s, mul_rn(lower, 1.0 - 1e-9))) return false;
    if (s.step_count <= s.warmup) return true;
    if (!(s.ewma_current >= s.ewma_previous)) return false;
    return rel_change_core(s.ewma_previous, s.ewma_current) >= delta;
}

// K2 body: one thread. Writes the flag word and the trace row; returns the word.
__device__ int signal_step_dev(ss_signal_state* st, double x, double delta, int32_t* word,
                                ss_trace_row* trace, int32_t cap) {
    ss_signal_state s = *st;
    int err = observe_core(&s, x);
    ss_trace_row row;
    row.grad_norm_sq = x;
    if (err) {
        st->error |= err;  // rest of the state unchanged (test_signal.py:72-76)
        row.ewma = s.ewma_current;
        row.delta_g = d_nan();
        row.step = static_cast<int32_t>(s.step_count);
        row.word = err;
    } else {
        *st = s;
        row.ewma = s.ewma_current;
        row.delta_g = s.last_delta;
        row.step = static_cast<int32_t>(s.step_count - 1);
        row.word = vote_core(&s, delta) ? SS_FLAG_SYNC : 0;
    }
    if (word) *word = row.word;
    if (trace && cap > 0) trace[row.step % cap] = row;
    return row.word;
}

// ----------------------------------------------------- memory helpers

// cache policies for the streaming update (selected per instantiation; 0 is the default):
//   0: ld/st .cs (evict-first)     1: plain ld/st
//   2: ld .L1::no_allocate.L2::256B prefetch, st .cs
//   3: like 2, gradient through the non-coherent path (ld.global.nc)
template <int CP>
__device__ __forceinline__ float4 ld_pol(const float* p) {
    if constexpr (CP == 1) {
        return *reinterpret_cast<const float4*>(p);
    } else if constexpr (CP >= 2) {
        float4 v;
        asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        return v;
    } else {
        return __ldcs(reinterpret_cast<const float4*>(p));
    }
}
template <int CP>
__device__ __forceinline__ float4 ld_pol_ro(const float* p) {
    if constexpr (CP == 3) {
        float4 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        return v;
    } else {
        return ld_pol<CP>(p);
    }
}
template <int CP>
__device__ __forceinline__ void st_pol(float* p, float4 v) {
    if constexpr (CP == 1) {
        *reinterpret_cast<float4*>(p) = v;
    } else {
        __stcs(reinterpret_cast<float4*>(p), v);
    }
}

__device__ __forceinline__ float4 ld_cs4(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_cs4(float* p, float4 v) {
    __stcs(reinterpret_cast<float4*>(p), v);
}

__device__ __forceinline__ double sq4(float4 v, double acc) {
    acc = fma(static_cast<double>(v.x), static_cast<double>(v.x), acc);
    acc = fma(static_cast<double>(v.y), static_cast<double>(v.y), acc);
    acc = fma(static_cast<double>(v.z), static_cast<double>(v.z), acc);
    acc = fma(static_cast<double>(v.w), static_cast<double>(v.w), acc);
    return acc;
}

__device__ __forceinline__ bool is_nan4(float4 v) {
    return (v.x != v.x) | (v.y != v.y) | (v.z != v.z) | (v.w != v.w);
}

// block sum; the value is valid in thread 0 only (fixed order => deterministic)
__device__ double block_sum(double v) {
    __shared__ double smem[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    v = (threadIdx.x < nw) ? smem[threadIdx.x] : 0.0;
    if (wid == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    __syncthreads();  // smem reusable by the caller afterwards
    return v;
}

struct Finish {
    void* ws;
    int block_offset;  // partial slot of blockIdx.x == 0 (multi-launch tables)
    int total_blocks;  // blocks over all launches feeding this reduction
    double* out;       // optional: ||g||^2
    ss_signal_state* st;  // optional: run K2 on the total
    double delta;
    int32_t* word;
    ss_trace_row* trace;
    int32_t cap;
};

// Deterministic two-pass finish inside the same launch.
__device__ void finish_norm(const Finish& f, double acc, VBlk vb) {
    __shared__ bool s_last;
    Workspace ws = ws_view(f.ws);
    double bsum = block_sum(acc);
    if (f.total_blocks == 1) {
        // the only block is the last one: no partials round trip (same value:
        // the two-pass sum of one partial and zeros is exact)
        if (threadIdx.x == 0) {
            if (f.out) *f.out = bsum;
            if (f.st) signal_step_dev(f.st, bsum, f.delta, f.word, f.trace, f.cap);
        }
        return;
    }
    if (threadIdx.x == 0) {
        ws.partials[f.block_offset + vb.bid] = bsum;
        __threadfence();
        unsigned int prev = atomicAdd(ws.counter, 1u);
        s_last = (prev == static_cast<unsigned int>(f.total_blocks - 1));
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double v = 0.0;
    for (int i = threadIdx.x; i < f.total_blocks; i += blockDim.x) v += __ldcg(ws.partials + i);
    v = block_sum(v);
    if (threadIdx.x == 0) {
        *ws.counter = 0u;  // self-reset: the next launch (or graph replay) starts clean
        if (f.out) *f.out = v;
        if (f.st) signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
    }
}
__device__ __forceinline__ void finish_norm(const Finish& f, double acc) { finish_norm(f, acc, hw_blk()); }

// ---------------------------------------------------------------- K1 pass

// this thread's fp64 partial of ||g||^2 over a grid-stride sweep
template <int U>
__device__ __forceinline__ double norm_pass(const float* __restrict__ g, int64_t n, int64_t head, VBlk vb) {
    const int64_t tid = static_cast<int64_t>(vb.bid) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(vb.n) * blockDim.x;
    double acc = 0.0;
    for (int64_t i = tid; i < head; i += stride) acc = fma((double)g[i], (double)g[i], acc);
    const float* gb = g + head;
    const int64_t nvec = (n - head) >> 2;
    int64_t i = tid;
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_cs4(gb + 4 * (i + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u) acc = sq4(v[u], acc);
    }
    for (; i < nvec; i += stride) acc = sq4(ld_cs4(gb + 4 * i), acc);
    for (int64_t j = head + 4 * nvec + tid; j < n; j += stride) acc = fma((double)g[j], (double)g[j], acc);
    return acc;
}
// Chunk c of C of the same sweep (the float4 vectors split into C contiguous
// ranges, each grid-strided; the head scalars go with chunk 0, the tail with
// chunk C - 1), accumulated onto acc.
template <int U>
__device__ __forceinline__ double norm_chunk(const float* __restrict__ g, int64_t n, int64_t head, VBlk vb, int c,
                                             int C, double acc) {
    const int64_t tid = static_cast<int64_t>(vb.bid) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(vb.n) * blockDim.x;
    const float* gb = g + head;
    const int64_t nvec = (n - head) >> 2;
    if (c == 0)
        for (int64_t i = tid; i < head; i += stride) acc = fma((double)g[i], (double)g[i], acc);
    const int64_t v0 = nvec * c / C, v1 = nvec * (c + 1) / C;
    int64_t i = v0 + tid;
    for (; i + (U - 1) * stride < v1; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_cs4(gb + 4 * (i + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u) acc = sq4(v[u], acc);
    }
    for (; i < v1; i += stride) acc = sq4(ld_cs4(gb + 4 * i), acc);
    if (c == C - 1)
        for (int64_t j = head + 4 * nvec + tid; j < n; j += stride) acc = fma((double)g[j], (double)g[j], acc);
    return acc;
}

template <int U>
__device__ __forceinline__ double norm_pass(const float* __restrict__ g, int64_t n, int64_t head) {
    return norm_pass<U>(g, n, head, hw_blk());
}

// ---------------------------------------------------------------- K3 / K13

struct SgdArgs {
    float* w;
    const float* g;
    float* m;
    int64_t n;
    int64_t head;  // leading scalars until the 16-byte boundary
    float lr, mu, damp, wd;
    int first;
    const int32_t* sync_word;
    float sync_scale;
};

template <bool MOM, bool NEST>
__device__ __forceinline__ void sgd_elem(float& w, float g, float& m, const SgdArgs& a, float s) {
    float d = fmaf(a.wd, w, g);
    if (MOM) {
        m = a.first ? d : fmaf(a.mu, m, (1.0f - a.damp) * d);
        d = NEST ? fmaf(a.mu, m, d) : m;
    }
    w = fmaf(-a.lr, d, w) * s;
}

// One streaming pass of the update over the whole buffer; returns this
// thread's fp64 partial of ||g||^2 (0 when NORM is false).
template <bool MOM, bool NEST, bool NORM, int U, int CP = 0>
__device__ __forceinline__ double sgd_pass(const SgdArgs& a_in, VBlk vb) {
    // a register copy: a_in may live in shared memory (colocated launch), and
    // stores through the generic w / m pointers would otherwise force reloads
    const SgdArgs a = a_in;
    const int64_t tid = static_cast<int64_t>(vb.bid) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(vb.n) * blockDim.x;
    float s = 1.0f;
    if (a.sync_word != nullptr) {
        const int word = __ldg(a.sync_word);
        // an error bit anywhere (NaN / negative norm on some rank): change nothing,
        // as the reference raises in observe before sgd_step (strategies.py:286, :383)
        if (word & ~SS_FLAG_SYNC) return 0.0;
        if (word & SS_FLAG_SYNC) s = a.sync_scale;
    }
    double acc = 0.0;
    float mdummy = 0.0f;
    for (int64_t i = tid; i < a.head; i += stride) {
        float w = a.w[i], g = a.g[i];
        float m = MOM ? a.m[i] : 0.0f;
        if (NORM) acc = fma((double)g, (double)g, acc);
        sgd_elem<MOM, NEST>(w, g, MOM ? m : mdummy, a, s);
        a.w[i] = w;
        if (MOM) a.m[i] = m;
    }
    float* wb = a.w + a.head;
    const float* gb = a.g + a.head;
    float* mb = MOM ? a.m + a.head : nullptr;
    const int64_t nvec = (a.n - a.head) >> 2;
    int64_t i = tid;
#ifndef SS_K13_INDEX_LOOP  // A/B build switch (tools/ab_build.sh)
    if constexpr (U == 1) {
        // pointer-bumped loop with a 32-bit trip count: fewer live 64-bit
        // values than index arithmetic (keeps the 3-stream momentum pass in
        // 64 registers without spills at 4 blocks x 256 threads per SM)
        if (i < nvec) {
            const int iters = static_cast<int>((nvec - 1 - i) / stride) + 1;
            const int64_t step = 4 * stride;
            const float* pg = gb + 4 * i;
            float* pw = wb + 4 * i;
            float* pm = MOM ? mb + 4 * i : nullptr;
            for (int it = 0; it < iters; ++it) {
                float4 gv = ld_pol_ro<CP>(pg), wv = ld_pol<CP>(pw);
                float4 mm = MOM ? ld_pol<CP>(pm) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (NORM) acc = sq4(gv, acc);
                sgd_elem<MOM, NEST>(wv.x, gv.x, mm.x, a, s);
                sgd_elem<MOM, NEST>(wv.y, gv.y, mm.y, a, s);
                sgd_elem<MOM, NEST>(wv.z, gv.z, mm.z, a, s);
                sgd_elem<MOM, NEST>(wv.w, gv.w, mm.w, a, s);
                st_pol<CP>(pw, wv);
                if (MOM) st_pol<CP>(pm, mm);
                pg += step;
                pw += step;
                if (MOM) pm += step;
            }
        }
    } else
#endif
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
        float4 gv[U], wv[U], mv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = 4 * (i + u * stride);
            gv[u] = ld_pol_ro<CP>(gb + k);
            wv[u] = ld_pol<CP>(wb + k);
            if (MOM) mv[u] = ld_pol<CP>(mb + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = 4 * (i + u * stride);
            if (NORM) acc = sq4(gv[u], acc);
            float4 mm = MOM ? mv[u] : make_float4(0.f, 0.f, 0.f, 0.f);
            sgd_elem<MOM, NEST>(wv[u].x, gv[u].x, mm.x, a, s);
            sgd_elem<MOM, NEST>(wv[u].y, gv[u].y, mm.y, a, s);
            sgd_elem<MOM, NEST>(wv[u].z, gv[u].z, mm.z, a, s);
            sgd_elem<MOM, NEST>(wv[u].w, gv[u].w, mm.w, a, s);
            st_pol<CP>(wb + k, wv[u]);
            if (MOM) st_pol<CP>(mb + k, mm);
        }
    }
#ifndef SS_K13_INDEX_LOOP
    if constexpr (U > 1)  // with U == 1 the loop above covers every vector
#endif
    {
        for (; i < nvec; i += stride) {
            const int64_t k = 4 * i;
            float4 gv = ld_cs4(gb + k), wv = ld_cs4(wb + k);
            float4 mm = MOM ? ld_cs4(mb + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (NORM) acc = sq4(gv, acc);
            sgd_elem<MOM, NEST>(wv.x, gv.x, mm.x, a, s);
            sgd_elem<MOM, NEST>(wv.y, gv.y, mm.y, a, s);
            sgd_elem<MOM, NEST>(wv.z, gv.z, mm.z, a, s);
            sgd_elem<MOM, NEST>(wv.w, gv.w, mm.w, a, s);
            st_cs4(wb + k, wv);
            if (MOM) st_cs4(mb + k, mm);
        }
    }
    for (int64_t j = a.head + 4 * nvec + tid; j < a.n; j += stride) {
        float w = a.w[j], g = a.g[j];
        float m = MOM ? a.m[j] : 0.0f;
        if (NORM) acc = fma((double)g, (double)g, acc);
        sgd_elem<MOM, NEST>(w, g, MOM ? m : mdummy, a, s);
        a.w[j] = w;
        if (MOM) a.m[j] = m;
    }
    return acc;
}
template <bool MOM, bool NEST, bool NORM, int U, int CP = 0>
__device__ __forceinline__ double sgd_pass(const SgdArgs& a) {
    return sgd_pass<MOM, NEST, NORM, U, CP>(a, hw_blk());
}

// The update over elements [e0, e1) by the threads of ONE block (tile work of
// the overlapped sync step). Requires 16-byte-aligned streams (head == 0) and
// e0 % 4 == 0; a scalar tail is handled when e1 is not a multiple of 4.
// NORM: also return this thread's fp64 partial of ||g||^2 over the range.
// NANF: return 1 when this thread met a NaN gradient element, else 0.
template <bool MOM, bool NEST, int U = 2, bool G_L2 = false, bool NORM = false, bool NANF = false>
__device__ __forceinline__ double sgd_block_range(const SgdArgs& a_in, int64_t e0, int64_t e1) {
    const SgdArgs a = a_in;  // register copy (see sgd_pass)
    // G_L2: read g through L2 only (it was just rewritten by peers over NVLink)
    // U vectors per stream in flight per thread: in the overlapped step only
    // part of the grid updates at a time, so each block needs more bytes in
    // flight than in the whole-grid K13 sweep (where U = 1 is best)
    const float s = 1.0f;
    double acc = 0.0;
    bool bad = false;
    const int64_t v0 = e0 >> 2, v1 = e1 >> 2;
    const int64_t bs = blockDim.x;
    int64_t i = v0 + threadIdx.x;
    for (; i + (U - 1) * bs < v1; i += U * bs) {
        float4 gv[U], wv[U], mv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = 4 * (i + u * bs);
            gv[u] = G_L2 ? __ldcg(reinterpret_cast<const float4*>(a.g + k)) : ld_cs4(a.g + k);
            wv[u] = ld_cs4(a.w + k);
            if (MOM) mv[u] = ld_cs4(a.m + k);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = 4 * (i + u * bs);
            if (NORM) acc = sq4(gv[u], acc);
            if (NANF) bad |= is_nan4(gv[u]);
            float4 mm = MOM ? mv[u] : make_float4(0.f, 0.f, 0.f, 0.f);
            sgd_elem<MOM, NEST>(wv[u].x, gv[u].x, mm.x, a, s);
            sgd_elem<MOM, NEST>(wv[u].y, gv[u].y, mm.y, a, s);
            sgd_elem<MOM, NEST>(wv[u].z, gv[u].z, mm.z, a, s);
            sgd_elem<MOM, NEST>(wv[u].w, gv[u].w, mm.w, a, s);
            st_cs4(a.w + k, wv[u]);
            if (MOM) st_cs4(a.m + k, mm);
        }
    }
    for (; i < v1; i += bs) {
        const int64_t k = 4 * i;
        float4 gv = G_L2 ? __ldcg(reinterpret_cast<const float4*>(a.g + k)) : ld_cs4(a.g + k);
        float4 wv = ld_cs4(a.w + k);
        float4 mm = MOM ? ld_cs4(a.m + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (NORM) acc = sq4(gv, acc);
        if (NANF) bad |= is_nan4(gv);
        sgd_elem<MOM, NEST>(wv.x, gv.x, mm.x, a, s);
        sgd_elem<MOM, NEST>(wv.y, gv.y, mm.y, a, s);
        sgd_elem<MOM, NEST>(wv.z, gv.z, mm.z, a, s);
        sgd_elem<MOM, NEST>(wv.w, gv.w, mm.w, a, s);
        st_cs4(a.w + k, wv);
        if (MOM) st_cs4(a.m + k, mm);
    }
    float mdummy = 0.0f;
    for (int64_t j = 4 * v1 + threadIdx.x; j < e1; j += bs) {
        float w = a.w[j], g = G_L2 ? __ldcg(a.g + j) : a.g[j];
        float m = MOM ? a.m[j] : 0.0f;
        if (NORM) acc = fma(static_cast<double>(g), static_cast<double>(g), acc);
        if (NANF) bad |= g != g;
        sgd_elem<MOM, NEST>(w, g, MOM ? m : mdummy, a, s);
        a.w[j] = w;
        if (MOM) a.m[j] = m;
    }
    if (NANF) return bad ? 1.0 : 0.0;
    return acc;
}

}  // namespace
