// host_util.cuh -- host-side launch helpers shared by the translation units
// of libselsync_b200.so (launch geometry, argument validation). Internal.
#pragma once

#include "device_core.cuh"

#include <cmath>
#include <cstdint>

namespace {

inline int sm_count_impl() {
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

inline int64_t grid_for(int64_t work_items, int per_thread, int resident) {
    int64_t want = (work_items + static_cast<int64_t>(kThreads) * per_thread - 1) /
                   (static_cast<int64_t>(kThreads) * per_thread);
    int64_t cap = static_cast<int64_t>(ss_internal::sm_count()) * resident;
    if (cap > kMaxGrid) cap = kMaxGrid;
    if (want > cap) want = cap;
    return want < 1 ? 1 : want;
}

// leading scalars until 16-byte alignment, or n (all scalar) if the streams
// do not share the same alignment phase
inline int64_t common_head(int64_t n, const void* a, const void* b, const void* c) {
    uintptr_t pa = reinterpret_cast<uintptr_t>(a);
    if ((pa & 3) != 0) return n;
    uintptr_t phase = pa & 15;
    if (b && (reinterpret_cast<uintptr_t>(b) & 15) != phase) return n;
    if (c && (reinterpret_cast<uintptr_t>(c) & 15) != phase) return n;
    int64_t head = static_cast<int64_t>(((16 - phase) & 15) >> 2);
    return head > n ? n : head;
}

inline int check_delta_impl(double delta) {
    if (!std::isfinite(delta) || delta < 0.0)
        return ss_internal::fail(SS_ERR_SIGNAL, "delta must be finite and >= 0, got %g", delta);
    return SS_OK;
}

inline int check_trace(ss_trace_row* trace, int32_t cap) {
    if (cap < 0 || (trace != nullptr && cap == 0))
        return ss_internal::fail(SS_ERR_CONFIG, "trace_cap must be > 0 when a trace ring is given, got %d", cap);
    return SS_OK;
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline int make_sgd_args(SgdArgs* a, float* w, const float* g, float* m, int64_t n, float lr, float mu,
                  float damp, float wd, int32_t nesterov, int32_t first, const int32_t* sync_word,
                  float sync_scale) {
    if (n < 0) return ss_internal::fail(SS_ERR_CONFIG, "n must be >= 0, got %lld", (long long)n);
    if (n > 0 && (!w || !g)) return ss_internal::fail(SS_ERR_CONFIG, "null parameter/gradient pointer");
    if (!(lr >= 0.0f)) return ss_internal::fail(SS_ERR_CONFIG, "learning rate must be non-negative, got %g", (double)lr);
    if (!(mu >= 0.0f)) return ss_internal::fail(SS_ERR_CONFIG, "momentum must be >= 0, got %g", (double)mu);
    if (!(wd >= 0.0f)) return ss_internal::fail(SS_ERR_CONFIG, "weight_decay must be >= 0, got %g", (double)wd);
    if (nesterov && (mu <= 0.0f || damp != 0.0f))
        return ss_internal::fail(SS_ERR_CONFIG, "Nesterov momentum requires a momentum and zero dampening");
    const bool mom = mu != 0.0f;
    if (mom && n > 0 && !m) return ss_internal::fail(SS_ERR_CONFIG, "momentum buffer required when momentum != 0");
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
