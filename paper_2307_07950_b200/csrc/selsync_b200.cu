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
#include "device_core.cuh"
#include "host_util.cuh"

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

// ---------------------------------------------------------------- K1

template <int U>
__global__ void __launch_bounds__(kThreads, 4) norm_kernel(const float* __restrict__ g, int64_t n,
                                                        int64_t head, Finish f) {
    pdl_wait();
    pdl_trigger();
    finish_norm(f, norm_pass<U>(g, n, head));
}

// ---------------------------------------------------------------- K2

__global__ void signal_kernel(ss_signal_state* st, const double* x, double delta, int32_t* word,
                              ss_trace_row* trace, int32_t cap) {
    signal_step_dev(st, *x, delta, word, trace, cap);
}

template <bool MOM, bool NEST, bool NORM, int U, int CP = 0>
__global__ void __launch_bounds__(kThreads, 4) sgd_kernel(SgdArgs a, Finish f) {
    pdl_wait();
    pdl_trigger();
    const double acc = sgd_pass<MOM, NEST, NORM, U, CP>(a);
    if (NORM) finish_norm(f, acc);
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

template <int U>
int launch_norm_u(const float* g, int64_t n, Finish f, void* stream, const char* what) {
    static const int resident = resident_blocks(norm_kernel<U>);
    const int64_t head = n ? common_head(n, g, nullptr, nullptr) : 0;
    const int grid = static_cast<int>(grid_for((n - head) / 4 + 1, U, resident));
    f.total_blocks = grid;
    (void)launch_ex(norm_kernel<U>, grid, kThreads, as_stream(stream), false, g, n, head, f);
    return check_launch(what);
}

// K1 unroll: 4 independent 16-byte loads in flight per thread (measured at
// P = 100M: U = 4 6.29-6.42 TB/s, the best of 1 / 2 / 4 / 8)
int launch_norm(const float* g, int64_t n, const Finish& f, void* stream, const char* what) {
    return launch_norm_u<kNormUnroll>(g, n, f, stream, what);
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
int sm_count() { return ::sm_count_impl(); }
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

int ss_sync_known_ahead(const ss_signal_state* st, double delta, int32_t* known_out) {
    if (!st || !known_out) return fail(SS_ERR_CONFIG, "null argument");
    int rc = check_delta_impl(delta);
    if (rc) return rc;
    *known_out = sync_known_ahead_core(st->step_count, st->warmup, delta, st->ewma_current) ? 1 : 0;
    return SS_OK;
}

int ss_sync_proven_early(const ss_signal_state* st, double lower, double delta, int32_t* proven_out) {
    if (!st || !proven_out) return fail(SS_ERR_CONFIG, "null argument");
    int rc = check_delta_impl(delta);
    if (rc) return rc;
    *proven_out = sync_proven_early_core(st, lower, delta) ? 1 : 0;
    return SS_OK;
}

int ss_workspace_bytes(int64_t* bytes) {
    if (!bytes) return fail(SS_ERR_CONFIG, "null output");
    *bytes = kWsBytes;
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
    (void)launch_ex(sgd_kernel<MOM, NEST, NORM, U, CP>, grid, kThreads, as_stream(stream), false, a, f);
    return check_launch(NORM ? "ss_update_norm_signal_f32" : "ss_sgd_update_f32");
}

// measured at P = 100M (round-1 sweep over unroll x cache policy): momentum
// (3 streams) U=1 6.40 TB/s vs U=2 5.92, U=4 5.67; plain (2 streams) U=2 6.23
// vs U=1 6.01; evict-first (.cs) loads/stores beat plain, L2::256B prefetch
// and the non-coherent gradient path
template <bool MOM>
constexpr int kSgdUnroll = MOM ? 1 : 2;

template <bool MOM, bool NEST, bool NORM>
int launch_sgd(const SgdArgs& a, const Finish& f0, void* stream) {
    return launch_sgd_v<MOM, NEST, NORM, kSgdUnroll<MOM>, 0>(a, f0, stream);
}

template <bool NORM>
int dispatch_sgd(const SgdArgs& a, const Finish& f, bool mom, bool nest, void* stream) {
    if (!mom) return launch_sgd<false, false, NORM>(a, f, stream);
    if (nest) return launch_sgd<true, true, NORM>(a, f, stream);
    return launch_sgd<true, false, NORM>(a, f, stream);
}



template <bool MOM, bool NEST>
void* k13_kernel_ptr() {
    return reinterpret_cast<void*>(sgd_kernel<MOM, NEST, true, kSgdUnroll<MOM>, 0>);
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

namespace ss_internal {
// the K13+K2 kernel of a prepared step (ss_step_plan_init) and its grid factor
void* k13_kernel(bool mom, bool nest, int* per_thread) {
    *per_thread = mom ? kSgdUnroll<true> : kSgdUnroll<false>;
    if (!mom) return k13_kernel_ptr<false, false>();
    return nest ? k13_kernel_ptr<true, true>() : k13_kernel_ptr<true, false>();
}
}  // namespace ss_internal
