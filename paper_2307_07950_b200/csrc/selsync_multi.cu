// selsync_multi.cu -- the SelSync update over a LIST of tensors (no flat buffer).
//
// For models whose parameters / gradients are separate allocations (the
// reference's ParamVector is always flat, model.py:54-66; a PyTorch model is
// not): K13 (sgd_step model.py:215-221 + ||g||^2 strategies.py:285) and K3
// over a pointer table, one logical launch per <= kMtUpd tensors. Blocks own
// contiguous ranges of the virtual concatenation of the tensors and walk the
// tensor segments inside their range (binary search for the first one); each
// segment streams 16-byte vectors when the three streams share an alignment
// phase, scalars otherwise. The fp64 partials of all launches meet in one
// deterministic finish (arrival counter spanning the launches), whose last
// block runs the signal step K2.

#include "selsync_b200.h"
#include "common.cuh"
#include "device_core.cuh"
#include "host_util.cuh"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

using ss_internal::check_launch;
using ss_internal::fail;

namespace {

constexpr int kMtUpd = 128;  // tensors per launch (kernel-parameter table)

struct UpdTable {
    float* w[kMtUpd];
    const float* g[kMtUpd];
    float* m[kMtUpd];
    int64_t start[kMtUpd + 1];
    int count;
    int64_t per_block;
};

template <bool MOM, bool NEST, bool NORM>
__device__ __forceinline__ double update_segment(float* w, const float* g, float* m, int64_t len,
                                                 const SgdArgs& a, float s, double acc) {
    // a common 16-byte phase for all streams -> scalar head, vector body, scalar tail
    const uintptr_t pw = reinterpret_cast<uintptr_t>(w), pg = reinterpret_cast<uintptr_t>(g);
    const uintptr_t pm = MOM ? reinterpret_cast<uintptr_t>(m) : pw;
    int64_t head = len;
    if ((pw & 3) == 0 && (pw & 15) == (pg & 15) && (pw & 15) == (pm & 15)) {
        head = static_cast<int64_t>(((16 - (pw & 15)) & 15) >> 2);
        if (head > len) head = len;
    }
    float mdummy = 0.0f;
    for (int64_t i = threadIdx.x; i < head; i += blockDim.x) {
        float wi = w[i], gi = g[i];
        float mi = MOM ? m[i] : 0.0f;
        if (NORM) acc = fma((double)gi, (double)gi, acc);
        sgd_elem<MOM, NEST>(wi, gi, MOM ? mi : mdummy, a, s);
        w[i] = wi;
        if (MOM) m[i] = mi;
    }
    const int64_t nvec = (len - head) >> 2;
    float* wb = w + head;
    const float* gb = g + head;
    float* mb = MOM ? m + head : nullptr;
    for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x) {
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
    for (int64_t j = head + 4 * nvec + threadIdx.x; j < len; j += blockDim.x) {
        float wi = w[j], gi = g[j];
        float mi = MOM ? m[j] : 0.0f;
        if (NORM) acc = fma((double)gi, (double)gi, acc);
        sgd_elem<MOM, NEST>(wi, gi, MOM ? mi : mdummy, a, s);
        w[j] = wi;
        if (MOM) m[j] = mi;
    }
    return acc;
}

template <bool MOM, bool NEST, bool NORM>
__global__ void __launch_bounds__(kThreads, 4) update_multi_kernel(UpdTable t, SgdArgs a, Finish f) {
    float s = 1.0f;
    if (a.sync_word != nullptr && (__ldg(a.sync_word) & SS_FLAG_SYNC)) s = a.sync_scale;
    const int64_t total = t.start[t.count];
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * t.per_block;
    const int64_t hi = lo + t.per_block < total ? lo + t.per_block : total;
    double acc = 0.0;
    if (lo < hi) {
        int b0 = 0, b1 = t.count - 1;  // first tensor with start[k + 1] > lo
        while (b0 < b1) {
            const int mid = (b0 + b1) >> 1;
            if (t.start[mid + 1] > lo) b1 = mid; else b0 = mid + 1;
        }
        for (int k = b0; k < t.count && t.start[k] < hi; ++k) {
            const int64_t s0 = lo > t.start[k] ? lo : t.start[k];
            const int64_t s1 = hi < t.start[k + 1] ? hi : t.start[k + 1];
            if (s1 > s0) {
                const int64_t off = s0 - t.start[k];
                acc = update_segment<MOM, NEST, NORM>(t.w[k] + off, t.g[k] + off, MOM ? t.m[k] + off : nullptr,
                                                      s1 - s0, a, s, acc);
            }
        }
    }
    if (NORM) finish_norm(f, acc);
}

template <bool MOM, bool NEST, bool NORM>
int launch_multi(float* const* w, const float* const* g, float* const* m, const int64_t* sizes, int32_t count,
                 const SgdArgs& a, Finish f, void* stream) {
    static const int resident = resident_blocks(update_multi_kernel<MOM, NEST, NORM>);
    const int n_groups = count == 0 ? 1 : (count + kMtUpd - 1) / kMtUpd;
    if (n_groups > 4096) return fail(SS_ERR_CONFIG, "too many tensors: %d", count);
    // pass 1: grids per group (total blocks feed one deterministic finish)
    static thread_local int grids[4096];
    static thread_local int64_t per_block[4096];
    int total_blocks = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
        int64_t tot = 0;
        for (int k = gi * kMtUpd; k < count && k < (gi + 1) * kMtUpd; ++k) tot += sizes[k];
        int grid = static_cast<int>(grid_for(tot / 4 + 1, 1, resident));
        if (total_blocks + grid > kMaxGrid) grid = 1;
        if (total_blocks + grid > kMaxGrid) return fail(SS_ERR_CONFIG, "too many tensor groups");
        int64_t pb = (tot + grid - 1) / grid;
        pb = ((pb + 1023) / 1024) * 1024;
        grids[gi] = grid;
        per_block[gi] = pb < 1024 ? 1024 : pb;
        total_blocks += grid;
    }
    f.total_blocks = total_blocks;
    int offset = 0;
    for (int gi = 0; gi < n_groups; ++gi) {
        UpdTable t;
        std::memset(&t, 0, sizeof(t));
        const int lo = gi * kMtUpd, hi = count < lo + kMtUpd ? count : lo + kMtUpd;
        t.count = hi - lo;
        t.start[0] = 0;
        for (int k = lo; k < hi; ++k) {
            t.w[k - lo] = w[k];
            t.g[k - lo] = g[k];
            t.m[k - lo] = MOM ? m[k] : nullptr;
            t.start[k - lo + 1] = t.start[k - lo] + sizes[k];
        }
        t.per_block = per_block[gi];
        Finish fg = f;
        fg.block_offset = offset;
        update_multi_kernel<MOM, NEST, NORM><<<grids[gi], kThreads, 0, static_cast<cudaStream_t>(stream)>>>(t, a, fg);
        const int rc = check_launch(NORM ? "ss_update_norm_signal_multi_f32" : "ss_sgd_update_multi_f32");
        if (rc) return rc;
        offset += grids[gi];
    }
    return SS_OK;
}

int check_table(float* const* w, const float* const* g, float* const* m, const int64_t* sizes, int32_t count,
                bool mom) {
    if (count < 1 || !w || !g || !sizes || (mom && !m)) return fail(SS_ERR_CONFIG, "bad tensor table");
    for (int k = 0; k < count; ++k) {
        if (sizes[k] < 0) return fail(SS_ERR_CONFIG, "negative size for tensor %d", k);
        if (sizes[k] > 0 && (!w[k] || !g[k] || (mom && !m[k])))
            return fail(SS_ERR_CONFIG, "null pointer for tensor %d", k);
    }
    return SS_OK;
}

template <bool NORM>
int dispatch_multi(float* const* w, const float* const* g, float* const* m, const int64_t* sizes, int32_t count,
                   const SgdArgs& a, const Finish& f, bool mom, bool nest, void* stream) {
    if (!mom) return launch_multi<false, false, NORM>(w, g, m, sizes, count, a, f, stream);
    if (nest) return launch_multi<true, true, NORM>(w, g, m, sizes, count, a, f, stream);
    return launch_multi<true, false, NORM>(w, g, m, sizes, count, a, f, stream);
}

}  // namespace

extern "C" {

int ss_sgd_update_multi_f32(float* const* w, const float* const* g, float* const* m, const int64_t* sizes,
                            int32_t count, float lr, float momentum, float dampening, float weight_decay,
                            int32_t nesterov, int32_t first_step, const int32_t* sync_word, float sync_scale,
                            void* stream) {
    SgdArgs a;
    // scalar validation through the flat-path helper (pointers checked per tensor below)
    int rc = make_sgd_args(&a, nullptr, nullptr, nullptr, 0, lr, momentum, dampening, weight_decay, nesterov,
                           first_step, sync_word, sync_scale);
    if (rc) return rc;
    const bool mom = momentum != 0.0f;
    rc = check_table(w, g, m, sizes, count, mom);
    if (rc) return rc;
    Finish f{nullptr, 0, 0, nullptr, nullptr, 0.0, nullptr, nullptr, 0};
    return dispatch_multi<false>(w, g, m, sizes, count, a, f, mom, nesterov != 0, stream);
}

int ss_update_norm_signal_multi_f32(float* const* w, const float* const* g, float* const* m, const int64_t* sizes,
                                    int32_t count, float lr, float momentum, float dampening, float weight_decay,
                                    int32_t nesterov, int32_t first_step, ss_signal_state* st, double delta,
                                    int32_t* word, ss_trace_row* trace, int32_t cap, void* ws, void* stream) {
    SgdArgs a;
    int rc = make_sgd_args(&a, nullptr, nullptr, nullptr, 0, lr, momentum, dampening, weight_decay, nesterov,
                           first_step, nullptr, 1.0f);
    if (rc) return rc;
    const bool mom = momentum != 0.0f;
    rc = check_table(w, g, m, sizes, count, mom);
    if (rc) return rc;
    if (!st || !ws) return fail(SS_ERR_CONFIG, "null state/workspace");
    rc = check_delta_impl(delta);
    if (rc) return rc;
    rc = check_trace(trace, cap);
    if (rc) return rc;
    Finish f{ws, 0, 0, nullptr, st, delta, word, trace, cap};
    return dispatch_multi<true>(w, g, m, sizes, count, a, f, mom, nesterov != 0, stream);
}

}  // extern "C"
