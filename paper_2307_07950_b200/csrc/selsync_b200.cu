// selsync_b200.cu -- sm_100a kernels + C-ABI for SelSync's per-step hot path.
//
// Path (reference: /root/reference/pkg/src/selsync):
//   K1  ||g||^2                 strategies.py:285        float(grad @ grad)
//   K2  EWMA / Delta / decide    signal.py:64-107         observe, relative_change, decide
//   K3  local update            model.py:215-221         sgd_step (+momentum, +weight decay)
//   K13 K3 with K1 fused, K2 in the finishing block (parameter aggregation order,
//       strategies.py:378-384: the local update lands before the vote)
//   replica mean / flag max     strategies.py:159-168, runtime.py:319-333 (simulated workers)
// The collectives (1-int allreduce-MAX, parameter allreduce) are NCCL calls
// issued by the host shim on the same stream; see DESIGN.md.
//
// All streaming kernels are HBM-bound: 128-bit vector loads/stores with
// evict-first cache hints, several independent 16-byte loads in flight per
// thread, grid = (#SMs x resident blocks) with a grid-stride loop so the whole
// buffer is covered by one wave. Norms accumulate in fp64 (squares of fp32
// values are exact in fp64) and finish deterministically: every block writes
// its partial, the last block to arrive (threadfence + arrival counter) sums
// the partials in a fixed order and, when asked, runs the signal step -- so
// K1+K2 (or K13+K2) is ONE launch and the flag word is on the device as soon
// as the kernel retires.

#include "selsync_b200.h"
#include "common.cuh"
#include "symm_device.cuh"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

namespace {

// ---------------------------------------------------------------- errors

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return SS_OK;
}

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

// K2 body: one thread. Writes the flag word and the trace row.
__device__ void signal_step_dev(ss_signal_state* st, double x, double delta, int32_t* word,
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
__device__ void finish_norm(const Finish& f, double acc) {
    __shared__ bool s_last;
    Workspace ws = ws_view(f.ws);
    double bsum = block_sum(acc);
    if (threadIdx.x == 0) {
        ws.partials[f.block_offset + blockIdx.x] = bsum;
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

// ---------------------------------------------------------------- K1

template <int U>
__global__ void __launch_bounds__(kThreads, 4) norm_kernel(const float* __restrict__ g, int64_t n,
                                                        int64_t head, Finish f) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
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
    finish_norm(f, acc);
}

// ---------------------------------------------------------------- K2

__global__ void signal_kernel(ss_signal_state* st, const double* x, double delta, int32_t* word,
                              ss_trace_row* trace, int32_t cap) {
    signal_step_dev(st, *x, delta, word, trace, cap);
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
__device__ __forceinline__ double sgd_pass(const SgdArgs& a) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    float s = 1.0f;
    if (a.sync_word != nullptr && (__ldg(a.sync_word) & SS_FLAG_SYNC)) s = a.sync_scale;
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
__global__ void __launch_bounds__(kThreads, 4) sgd_kernel(SgdArgs a, Finish f) {
    const double acc = sgd_pass<MOM, NEST, NORM, U, CP>(a);
    if (NORM) finish_norm(f, acc);
}

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

// ------------------------------------------------- multi-tensor K1 (+K2)

struct MtTable {
    const float* ptr[kMtMax];
    int64_t start[kMtMax + 1];  // prefix sums over the virtual concatenation
    int count;
    int64_t per_block;
};

__device__ __forceinline__ double sq_segment(const float* p, int64_t len, double acc) {
    // scalar head to the 16-byte boundary, block-strided float4 body, scalar tail
    int64_t head = (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15;
    head = (head & 3) ? len : head >> 2;  // 4-byte-misaligned floats: all scalar
    if (head > len) head = len;
    for (int64_t i = threadIdx.x; i < head; i += blockDim.x) acc = fma((double)p[i], (double)p[i], acc);
    const float* b = p + head;
    const int64_t nvec = (len - head) >> 2;
    int64_t i = threadIdx.x;
    for (; i + 3 * blockDim.x < nvec; i += 4 * blockDim.x) {
        float4 v0 = ld_cs4(b + 4 * i), v1 = ld_cs4(b + 4 * (i + blockDim.x));
        float4 v2 = ld_cs4(b + 4 * (i + 2 * blockDim.x)), v3 = ld_cs4(b + 4 * (i + 3 * blockDim.x));
        acc = sq4(v0, acc);
        acc = sq4(v1, acc);
        acc = sq4(v2, acc);
        acc = sq4(v3, acc);
    }
    for (; i < nvec; i += blockDim.x) acc = sq4(ld_cs4(b + 4 * i), acc);
    for (int64_t j = head + 4 * nvec + threadIdx.x; j < len; j += blockDim.x)
        acc = fma((double)p[j], (double)p[j], acc);
    return acc;
}

__global__ void __launch_bounds__(kThreads) norm_multi_kernel(MtTable t, Finish f) {
    const int64_t total = t.start[t.count];
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * t.per_block;
    const int64_t hi = lo + t.per_block < total ? lo + t.per_block : total;
    double acc = 0.0;
    if (lo < hi) {
        int a = 0, b = t.count - 1;  // first tensor with start[k+1] > lo
        while (a < b) {
            int mid = (a + b) >> 1;
            if (t.start[mid + 1] > lo) b = mid; else a = mid + 1;
        }
        for (int k = a; k < t.count && t.start[k] < hi; ++k) {
            const int64_t s0 = lo > t.start[k] ? lo : t.start[k];
            const int64_t s1 = hi < t.start[k + 1] ? hi : t.start[k + 1];
            if (s1 > s0) acc = sq_segment(t.ptr[k] + (s0 - t.start[k]), s1 - s0, acc);
        }
    }
    finish_norm(f, acc);
}

// ------------------------------------------------- simulated workers

struct PtrTable {
    float* p[kMaxReplicas];
};

template <bool VEC, bool BCAST>
__global__ void __launch_bounds__(kThreads, 4) mean_kernel(PtrTable t, int count, int64_t n, float* out,
                                                        bool divide) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const float fc = divide ? static_cast<float>(count) : 1.0f;
    if (VEC) {
        const int64_t nvec = n >> 2;
        for (int64_t i = tid; i < nvec; i += stride) {
            float4 acc = ld_cs4(t.p[0] + 4 * i);
            for (int r = 1; r < count; ++r) {
                float4 v = ld_cs4(t.p[r] + 4 * i);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
            acc.x /= fc; acc.y /= fc; acc.z /= fc; acc.w /= fc;
            if (BCAST) {
                for (int r = 0; r < count; ++r) st_cs4(t.p[r] + 4 * i, acc);
            } else {
                st_cs4(out + 4 * i, acc);
            }
        }
        for (int64_t j = 4 * nvec + tid; j < n; j += stride) {
            float acc1 = t.p[0][j];
            for (int r = 1; r < count; ++r) acc1 += t.p[r][j];
            acc1 /= fc;
            if (BCAST) { for (int r = 0; r < count; ++r) t.p[r][j] = acc1; } else { out[j] = acc1; }
        }
    } else {
        for (int64_t j = tid; j < n; j += stride) {
            float acc1 = t.p[0][j];
            for (int r = 1; r < count; ++r) acc1 += t.p[r][j];
            acc1 /= fc;
            if (BCAST) { for (int r = 0; r < count; ++r) t.p[r][j] = acc1; } else { out[j] = acc1; }
        }
    }
}

struct WordTable {
    int32_t* p[kMaxReplicas];
};

__global__ void flag_max_kernel(WordTable t, int count) {
    int32_t m = t.p[0][0];
    for (int r = 1; r < count; ++r) m = t.p[r][0] > m ? t.p[r][0] : m;
    for (int r = 0; r < count; ++r) t.p[r][0] = m;
}

// ------------------------------------------------- launch geometry

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cache[dev] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        cache[dev] = v;
    }
    return cache[dev];
}

template <typename K>
int resident_blocks(K kernel) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b <= 0) b = 4;
    return b;
}

int64_t grid_for(int64_t work_items, int per_thread, int resident) {
    int64_t want = (work_items + static_cast<int64_t>(kThreads) * per_thread - 1) /
                   (static_cast<int64_t>(kThreads) * per_thread);
    int64_t cap = static_cast<int64_t>(sm_count()) * resident;
    if (cap > kMaxGrid) cap = kMaxGrid;
    if (want > cap) want = cap;
    return want < 1 ? 1 : want;
}

// leading scalars until 16-byte alignment, or n (all scalar) if the streams
// do not share the same alignment phase
int64_t common_head(int64_t n, const void* a, const void* b, const void* c) {
    uintptr_t pa = reinterpret_cast<uintptr_t>(a);
    if ((pa & 3) != 0) return n;
    uintptr_t phase = pa & 15;
    if (b && (reinterpret_cast<uintptr_t>(b) & 15) != phase) return n;
    if (c && (reinterpret_cast<uintptr_t>(c) & 15) != phase) return n;
    int64_t head = static_cast<int64_t>(((16 - phase) & 15) >> 2);
    return head > n ? n : head;
}

int check_delta_impl(double delta) {
    if (!std::isfinite(delta) || delta < 0.0)
        return fail(SS_ERR_SIGNAL, "delta must be finite and >= 0, got %g", delta);
    return SS_OK;
}

int check_trace(ss_trace_row* trace, int32_t cap) {
    if (cap < 0 || (trace != nullptr && cap == 0))
        return fail(SS_ERR_CONFIG, "trace_cap must be > 0 when a trace ring is given, got %d", cap);
    return SS_OK;
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

template <int U>
int launch_norm_u(const float* g, int64_t n, Finish f, void* stream, const char* what) {
    static const int resident = resident_blocks(norm_kernel<U>);
    const int64_t head = n ? common_head(n, g, nullptr, nullptr) : 0;
    const int grid = static_cast<int>(grid_for((n - head) / 4 + 1, U, resident));
    f.total_blocks = grid;
    norm_kernel<U><<<grid, kThreads, 0, as_stream(stream)>>>(g, n, head, f);
    return check_launch(what);
}

// SS_NORM_UNROLL overrides the K1 unroll for tuning sweeps
int launch_norm(const float* g, int64_t n, const Finish& f, void* stream, const char* what) {
    static int u = -1;
    if (u < 0) {
        const char* e = getenv("SS_NORM_UNROLL");
        u = e ? atoi(e) : 0;
    }
    switch (u) {
        case 1: return launch_norm_u<1>(g, n, f, stream, what);
        case 2: return launch_norm_u<2>(g, n, f, stream, what);
        case 4: return launch_norm_u<4>(g, n, f, stream, what);
        case 8: return launch_norm_u<8>(g, n, f, stream, what);
        default: return launch_norm_u<kNormUnroll>(g, n, f, stream, what);
    }
}

}  // namespace

namespace ss_internal {
int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
int check_launch(const char* what) { return ::check_launch(what); }
int sm_count() { return ::sm_count(); }
}  // namespace ss_internal

// =================================================================== C-ABI

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }
const char* ss_last_error(void) { return g_err; }
int ss_signal_state_size(void) { return static_cast<int>(sizeof(ss_signal_state)); }
int ss_trace_row_size(void) { return static_cast<int>(sizeof(ss_trace_row)); }

int ss_default_smoothing(int32_t n_workers, double* out) {
    if (!out) return fail(SS_ERR_CONFIG, "null output");
    if (n_workers < 1) return fail(SS_ERR_CONFIG, "n_workers must be positive, got %d", n_workers);
    if (n_workers == 1) { *out = 0.05; return SS_OK; }
    double v = static_cast<double>(n_workers) / 100.0;
    *out = v < 0.01 ? 0.01 : (v > 1.0 ? 1.0 : v);
    return SS_OK;
}

int ss_check_delta(double delta) { return check_delta_impl(delta); }

int ss_signal_init(ss_signal_state* st, double smoothing, int32_t warmup) {
    if (!st) return fail(SS_ERR_CONFIG, "null state");
    if (!(smoothing > 0.0 && smoothing <= 1.0))
        return fail(SS_ERR_SIGNAL, "smoothing must be in (0, 1], got %g", smoothing);
    if (warmup < 1) return fail(SS_ERR_SIGNAL, "warmup must be >= 1, got %d", warmup);
    std::memset(st, 0, sizeof(*st));
    st->smoothing = smoothing;
    st->warmup = warmup;
    st->last_delta = d_nan();
    return SS_OK;
}

int ss_signal_observe(ss_signal_state* st, double x) {
    if (!st) return fail(SS_ERR_CONFIG, "null state");
    ss_signal_state s = *st;
    int err = observe_core(&s, x);
    if (err & SS_FLAG_ERR_NAN) return fail(SS_ERR_SIGNAL, "observed a NaN gradient norm");
    if (err & SS_FLAG_ERR_NEG) return fail(SS_ERR_SIGNAL, "squared norm cannot be negative, got %g", x);
    *st = s;
    return SS_OK;
}

int ss_relative_change(const ss_signal_state* st, double* out) {
    if (!st || !out) return fail(SS_ERR_CONFIG, "null argument");
    if (st->step_count < 2) return fail(SS_ERR_SIGNAL, "relative change needs at least two observations");
    *out = rel_change_core(st->ewma_previous, st->ewma_current);
    return SS_OK;
}

int ss_decide(const ss_signal_state* st, double delta, int32_t* sync_out) {
    if (!st || !sync_out) return fail(SS_ERR_CONFIG, "null argument");
    int rc = check_delta_impl(delta);
    if (rc) return rc;
    if (st->step_count < 1) return fail(SS_ERR_SIGNAL, "decide called before any observation");
    *sync_out = vote_core(st, delta);
    return SS_OK;
}

int ss_workspace_bytes(int64_t* bytes) {
    if (!bytes) return fail(SS_ERR_CONFIG, "null output");
    *bytes = kWsHeader + static_cast<int64_t>(sizeof(double)) * kMaxGrid;
    return SS_OK;
}

int ss_workspace_reset(void* ws, void* stream) {
    if (!ws) return fail(SS_ERR_CONFIG, "null workspace");
    int64_t bytes = 0;
    ss_workspace_bytes(&bytes);
    if (cudaMemsetAsync(ws, 0, static_cast<size_t>(bytes), as_stream(stream)) != cudaSuccess)
        return check_launch("ss_workspace_reset");
    return SS_OK;
}

int ss_norm_sq_f32(const float* g, int64_t n, double* out, void* ws, void* stream) {
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0, got %lld", (long long)n);
    if ((n > 0 && !g) || !out || !ws) return fail(SS_ERR_CONFIG, "null pointer argument");
    Finish f{ws, 0, 0, out, nullptr, 0.0, nullptr, nullptr, 0};
    return launch_norm(g, n, f, stream, "ss_norm_sq_f32");
}

int ss_norm_sq_multi_f32(const float* const* ptrs, const int64_t* sizes, int32_t count, double* out,
                         ss_signal_state* st, double delta, int32_t* word, ss_trace_row* trace,
                         int32_t cap, void* ws, void* stream) {
    if (count < 0 || (count > 0 && (!ptrs || !sizes)) || !ws)
        return fail(SS_ERR_CONFIG, "bad tensor table");
    if (st) {
        int rc = check_delta_impl(delta);
        if (rc) return rc;
        rc = check_trace(trace, cap);
        if (rc) return rc;
    }
    static const int resident = resident_blocks(norm_multi_kernel);
    // launch plan: groups of <= kMtMax tensors, each with its own grid; the
    // arrival counter spans all of them so only the final group finishes
    int n_groups = count == 0 ? 1 : (count + kMtMax - 1) / kMtMax;
    int grids[1024];
    if (n_groups > 1024) return fail(SS_ERR_CONFIG, "too many tensors: %d", count);
    int64_t per_block[1024];
    int total_blocks = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
        int64_t tot = 0;
        for (int k = gi * kMtMax; k < count && k < (gi + 1) * kMtMax; ++k) {
            if (sizes[k] < 0 || (sizes[k] > 0 && !ptrs[k])) return fail(SS_ERR_CONFIG, "bad tensor %d", k);
            tot += sizes[k];
        }
        int grid = static_cast<int>(grid_for(tot / 4 + 1, 4, resident));
        if (total_blocks + grid > kMaxGrid) grid = 1;
        if (total_blocks + grid > kMaxGrid) return fail(SS_ERR_CONFIG, "too many tensor groups");
        int64_t pb = (tot + grid - 1) / grid;
        pb = ((pb + 1023) / 1024) * 1024;
        if (pb < 1024) pb = 1024;
        grids[gi] = grid;
        per_block[gi] = pb;
        total_blocks += grid;
    }
    int offset = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
        MtTable t;
        std::memset(&t, 0, sizeof(t));
        int lo = gi * kMtMax;
        int hi = count < lo + kMtMax ? count : lo + kMtMax;
        t.count = hi - lo;
        t.start[0] = 0;
        for (int k = lo; k < hi; ++k) {
            t.ptr[k - lo] = ptrs[k];
            t.start[k - lo + 1] = t.start[k - lo] + sizes[k];
        }
        t.per_block = per_block[gi];
        Finish f{ws, offset, total_blocks, out, st, delta, word, trace, cap};
        norm_multi_kernel<<<grids[gi], kThreads, 0, as_stream(stream)>>>(t, f);
        int rc = check_launch("ss_norm_sq_multi_f32");
        if (rc) return rc;
        offset += grids[gi];
    }
    return SS_OK;
}

int ss_signal_step(ss_signal_state* st, const double* x, double delta, int32_t* word,
                   ss_trace_row* trace, int32_t cap, void* stream) {
    if (!st || !x) return fail(SS_ERR_CONFIG, "null pointer argument");
    int rc = check_delta_impl(delta);
    if (rc) return rc;
    rc = check_trace(trace, cap);
    if (rc) return rc;
    signal_kernel<<<1, 1, 0, as_stream(stream)>>>(st, x, delta, word, trace, cap);
    return check_launch("ss_signal_step");
}

int ss_norm_signal_f32(const float* g, int64_t n, ss_signal_state* st, double delta, int32_t* word,
                       ss_trace_row* trace, int32_t cap, void* ws, void* stream) {
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0, got %lld", (long long)n);
    if ((n > 0 && !g) || !st || !ws) return fail(SS_ERR_CONFIG, "null pointer argument");
    int rc = check_delta_impl(delta);
    if (rc) return rc;
    rc = check_trace(trace, cap);
    if (rc) return rc;
    Finish f{ws, 0, 0, nullptr, st, delta, word, trace, cap};
    return launch_norm(g, n, f, stream, "ss_norm_signal_f32");
}

}  // extern "C"

namespace {

template <bool MOM, bool NEST, bool NORM, int U, int CP>
int launch_sgd_v(const SgdArgs& a, const Finish& f0, void* stream) {
    static const int resident = resident_blocks(sgd_kernel<MOM, NEST, NORM, U, CP>);
    const int grid = static_cast<int>(grid_for((a.n - a.head) / 4 + 1, U, resident));
    Finish f = f0;
    f.total_blocks = grid;
    sgd_kernel<MOM, NEST, NORM, U, CP><<<grid, kThreads, 0, as_stream(stream)>>>(a, f);
    return check_launch(NORM ? "ss_update_norm_signal_f32" : "ss_sgd_update_f32");
}

// SS_SGD_VARIANT="<cp><u>" (e.g. "21") overrides the cache policy / unroll of
// the momentum K13 kernel for tuning sweeps (tools/sgd_sweep.py); unset = default
// measured at P = 100M (tools/sgd_sweep.py): momentum (3 streams) U=1 6.40 TB/s vs U=2 5.92,
// U=4 5.67; plain (2 streams) U=2 6.23 vs U=1 6.01
template <bool MOM>
constexpr int kSgdUnroll = MOM ? 1 : 2;

int sgd_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("SS_SGD_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <bool MOM, bool NEST, bool NORM>
int launch_sgd(const SgdArgs& a, const Finish& f0, void* stream) {
    if constexpr (!NEST) {
        switch (sgd_variant()) {
            case 1: return launch_sgd_v<MOM, NEST, NORM, 1, 0>(a, f0, stream);
            case 4: return launch_sgd_v<MOM, NEST, NORM, 4, 0>(a, f0, stream);
            case 11: return launch_sgd_v<MOM, NEST, NORM, 1, 1>(a, f0, stream);
            case 12: return launch_sgd_v<MOM, NEST, NORM, 2, 1>(a, f0, stream);
            case 14: return launch_sgd_v<MOM, NEST, NORM, 4, 1>(a, f0, stream);
            case 21: return launch_sgd_v<MOM, NEST, NORM, 1, 2>(a, f0, stream);
            case 22: return launch_sgd_v<MOM, NEST, NORM, 2, 2>(a, f0, stream);
            case 24: return launch_sgd_v<MOM, NEST, NORM, 4, 2>(a, f0, stream);
            case 31: return launch_sgd_v<MOM, NEST, NORM, 1, 3>(a, f0, stream);
            case 32: return launch_sgd_v<MOM, NEST, NORM, 2, 3>(a, f0, stream);
            case 34: return launch_sgd_v<MOM, NEST, NORM, 4, 3>(a, f0, stream);
            case 2: return launch_sgd_v<MOM, NEST, NORM, 2, 0>(a, f0, stream);
            default: break;
        }
    }
    return launch_sgd_v<MOM, NEST, NORM, kSgdUnroll<MOM>, 0>(a, f0, stream);
}

template <bool NORM>
int dispatch_sgd(const SgdArgs& a, const Finish& f, bool mom, bool nest, void* stream) {
    if (!mom) return launch_sgd<false, false, NORM>(a, f, stream);
    if (nest) return launch_sgd<true, true, NORM>(a, f, stream);
    return launch_sgd<true, false, NORM>(a, f, stream);
}

int make_sgd_args(SgdArgs* a, float* w, const float* g, float* m, int64_t n, float lr, float mu,
                  float damp, float wd, int32_t nesterov, int32_t first, const int32_t* sync_word,
                  float sync_scale) {
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0, got %lld", (long long)n);
    if (n > 0 && (!w || !g)) return fail(SS_ERR_CONFIG, "null parameter/gradient pointer");
    if (!(lr >= 0.0f)) return fail(SS_ERR_CONFIG, "learning rate must be non-negative, got %g", (double)lr);
    if (!(mu >= 0.0f)) return fail(SS_ERR_CONFIG, "momentum must be >= 0, got %g", (double)mu);
    if (!(wd >= 0.0f)) return fail(SS_ERR_CONFIG, "weight_decay must be >= 0, got %g", (double)wd);
    if (nesterov && (mu <= 0.0f || damp != 0.0f))
        return fail(SS_ERR_CONFIG, "Nesterov momentum requires a momentum and zero dampening");
    const bool mom = mu != 0.0f;
    if (mom && n > 0 && !m) return fail(SS_ERR_CONFIG, "momentum buffer required when momentum != 0");
    a->w = w;
    a->g = g;
    a->m = mom ? m : nullptr;
    a->n = n;
    a->head = n ? common_head(n, g, w, mom ? m : nullptr) : 0;
    a->lr = lr;
    a->mu = mu;
    a->damp = damp;
    a->wd = wd;
    a->first = first ? 1 : 0;
    a->sync_word = sync_word;
    a->sync_scale = sync_scale;
    return SS_OK;
}

}  // namespace

extern "C" {

int ss_sgd_update_f32(float* w, const float* g, float* m, int64_t n, float lr, float momentum,
                      float dampening, float weight_decay, int32_t nesterov, int32_t first_step,
                      const int32_t* sync_word, float sync_scale, void* stream) {
    SgdArgs a;
    int rc = make_sgd_args(&a, w, g, m, n, lr, momentum, dampening, weight_decay, nesterov,
                           first_step, sync_word, sync_scale);
    if (rc) return rc;
    Finish f{nullptr, 0, 0, nullptr, nullptr, 0.0, nullptr, nullptr, 0};
    return dispatch_sgd<false>(a, f, momentum != 0.0f, nesterov != 0, stream);
}

int ss_update_norm_signal_f32(float* w, const float* g, float* m, int64_t n, float lr, float momentum,
                              float dampening, float weight_decay, int32_t nesterov,
                              int32_t first_step, ss_signal_state* st, double delta, int32_t* word,
                              ss_trace_row* trace, int32_t cap, void* ws, void* stream) {
    SgdArgs a;
    int rc = make_sgd_args(&a, w, g, m, n, lr, momentum, dampening, weight_decay, nesterov,
                           first_step, nullptr, 1.0f);
    if (rc) return rc;
    if (!st || !ws) return fail(SS_ERR_CONFIG, "null state/workspace");
    rc = check_delta_impl(delta);
    if (rc) return rc;
    rc = check_trace(trace, cap);
    if (rc) return rc;
    Finish f{ws, 0, 0, nullptr, st, delta, word, trace, cap};
    return dispatch_sgd<true>(a, f, momentum != 0.0f, nesterov != 0, stream);
}

}  // extern "C"

namespace {
int replica_reduce(float* const* bufs, int32_t count, int64_t n, bool divide, void* stream) {
    if (count < 1 || count > kMaxReplicas || !bufs)
        return fail(SS_ERR_CONFIG, "replica count must be in [1, %d], got %d", kMaxReplicas, count);
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0");
    if (n == 0 || count == 1) return SS_OK;
    PtrTable t;
    bool vec = true;
    for (int r = 0; r < count; ++r) {
        if (!bufs[r]) return fail(SS_ERR_CONFIG, "null replica buffer %d", r);
        t.p[r] = bufs[r];
        vec = vec && (reinterpret_cast<uintptr_t>(bufs[r]) & 15) == 0;
    }
    static const int res_v = resident_blocks(mean_kernel<true, true>);
    const int grid = static_cast<int>(grid_for(n / 4 + 1, 1, res_v));
    if (vec) mean_kernel<true, true><<<grid, kThreads, 0, as_stream(stream)>>>(t, count, n, nullptr, divide);
    else mean_kernel<false, true><<<grid, kThreads, 0, as_stream(stream)>>>(t, count, n, nullptr, divide);
    return check_launch(divide ? "ss_replica_average_f32" : "ss_replica_sum_f32");
}
}  // namespace

extern "C" {

int ss_replica_average_f32(float* const* bufs, int32_t count, int64_t n, void* stream) {
    return replica_reduce(bufs, count, n, true, stream);
}

int ss_replica_sum_f32(float* const* bufs, int32_t count, int64_t n, void* stream) {
    return replica_reduce(bufs, count, n, false, stream);
}

int ss_mean_f32(const float* const* bufs, int32_t count, int64_t n, float* out, void* stream) {
    if (count < 1 || count > kMaxReplicas || !bufs || (n > 0 && !out))
        return fail(SS_ERR_CONFIG, "bad mean arguments (count=%d)", count);
    if (n < 0) return fail(SS_ERR_CONFIG, "n must be >= 0");
    if (n == 0) return SS_OK;
    PtrTable t;
    bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (int r = 0; r < count; ++r) {
        if (!bufs[r]) return fail(SS_ERR_CONFIG, "null buffer %d", r);
        t.p[r] = const_cast<float*>(bufs[r]);
        vec = vec && (reinterpret_cast<uintptr_t>(bufs[r]) & 15) == 0;
    }
    static const int res_v = resident_blocks(mean_kernel<true, false>);
    const int grid = static_cast<int>(grid_for(n / 4 + 1, 1, res_v));
    if (vec) mean_kernel<true, false><<<grid, kThreads, 0, as_stream(stream)>>>(t, count, n, out, true);
    else mean_kernel<false, false><<<grid, kThreads, 0, as_stream(stream)>>>(t, count, n, out, true);
    return check_launch("ss_mean_f32");
}

int ss_replica_flag_max_i32(int32_t* const* words, int32_t count, void* stream) {
    if (count < 1 || count > kMaxReplicas || !words)
        return fail(SS_ERR_CONFIG, "replica count must be in [1, %d], got %d", kMaxReplicas, count);
    WordTable t;
    for (int r = 0; r < count; ++r) {
        if (!words[r]) return fail(SS_ERR_CONFIG, "null flag word %d", r);
        t.p[r] = words[r];
    }
    flag_max_kernel<<<1, 1, 0, as_stream(stream)>>>(t, count);
    return check_launch("ss_replica_flag_max_i32");
}

}  // extern "C"

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
    int avg_grid = sm_count() * avg_resident;
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
