// selsync_step.cu -- the whole SelSync step from ONE host launch.
//
// Reference path (/root/reference/pkg/src/selsync): _selsync_step
// (strategies.py:369-403) with the parameter server's flag relay
// (runtime.py:319-333) and mean round (runtime.py:275-294).
//
// step_kernel (one host launch per step) runs one of two orders, chosen on
// the device so every rank takes the same one:
//
//  update first (order 0): K13 -- update + ||g||^2 over the whole buffer; the
//     last block to arrive reduces the partials, runs K2, posts its vote to
//     every peer's signal slot and waits for the N votes (C1: MAX = OR), then
//     broadcasts the agreed word to the other blocks of the (one-wave) grid.
//     On sync all blocks run the NVLink mean of this rank's shard with the 1/N
//     in the epilogue (C2) + end barrier; on local steps they exit.
//     20P HBM bytes; a sync step pays update + mean back to back.
//
//  norm first (order 1): ONE ticketed pass of the same launch: first the ||g||^2 tiles (4P; the block that finishes the last
//     one runs K2 and posts the vote), then groups of N update tiles and one
//     mean ticket for a tile this rank owns (tile t belongs to rank t mod N)
//     that was updated `lag` groups earlier. A rank announces a finished
//     update tile by a remote atomic add on the owner's counter; a mean ticket
//     waits for the agreed vote (a no-op on local steps) and for all N counts.
//     Updates start while the vote is still in flight, and on sync steps the
//     HBM-bound update overlaps the NVLink-bound mean tile by tile. Tickets
//     only wait on earlier tickets, so the pass cannot deadlock.
//
//  adaptive (order 2): the last block keeps, per context of the previous two
//     agreed decisions, an EWMA of the decision that followed; the next step
//     uses order 1 when the prediction for the current context is >= threshold.
//
//  known sync (orders 1 and 2, with tile_norm): when the step is sync whatever
//     ||g||^2 turns out to be (warmup, or delta == 0), the ticketed pass runs
//     without the norm sweep and without waiting for the vote: each update
//     tile also yields its ||g||^2 partial, the block finishing the last tile
//     reduces them in tile order, runs K2 and posts the vote (still exchanged,
//     for the trace, the EWMA and NaN error bits); the mean overlaps the
//     update from the first tiles on. 20P HBM bytes instead of 24P.
//
//  All orders compute identical parameters (same per-element arithmetic).

#include "selsync_b200.h"
#include "common.cuh"
#include "device_core.cuh"
#include "host_util.cuh"
#include "symm_device.cuh"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

using ss_internal::check_launch;
using ss_internal::fail;

namespace {

struct OverlapArgs {
    uint32_t* cnt[kMaxRanks];  // per-rank tile arrival counters, indexed by tile
    uint32_t* epoch;
    float* predictor;          // 5 floats: P(sync) per 2-decision context + the context
    int mode;
    float threshold;
    int64_t tile;
    int64_t n_tiles;
    int lag;                   // groups between an update ticket and the owner's mean ticket
    int early;                 // exact early vote enabled (norm-first orders without the known pass)
    unsigned long long* ticket;
    uint64_t* dbg;             // optional per-ticket timeline: {kind << 48 | tile, t0, t_ready, t_end}
    int64_t dbg_cap;
    double* tile_norm;         // known-sync pass: ||g||^2 partial per tile (NULL: pass disabled)
    unsigned int* started;     // blocks that took this launch's order snapshot (workspace, self-resetting)
    double* running;           // early vote: running sum of the block partials (workspace, self-resetting)
    uint64_t* early_posted;    // early vote: seq of the last step this rank posted an early sync tag for
};

// A/B build switches of the small-P latency study (tools/small_p_probe.py):
// SS_VOTE_FENCE=1 restores a system fence before the vote posts. It is not
// needed: the posts are st.release.sys, and the blocks' updates reach the
// last block through the gpu-scope arrival counter (fence + atomic, atomic +
// fence), and causality order is transitive across the two scopes (measured:
// -1 to -1.5 us per step at N = 2, P = 1M-16M);
// SS_STEP_PER_THREAD = float4 vectors per thread (per stream) below which the
// step grid shrinks (small P: 244 instead of 592 blocks at 1M, -1.5 us per
// local step at N = 2; one full wave from 4M up); SS_DECIDED_SLEEP = ns
// between polls of the decision word
#ifndef SS_VOTE_FENCE
#define SS_VOTE_FENCE 0
#endif
#ifndef SS_STEP_PER_THREAD
#define SS_STEP_PER_THREAD 4
#endif
#ifndef SS_DECIDED_SLEEP
#define SS_DECIDED_SLEEP 256
#endif
__device__ __forceinline__ void vote_fence() {
#if SS_VOTE_FENCE
    __threadfence_system();
#endif
}

#ifndef SS_LAG_SCALE
#define SS_LAG_SCALE 1
#endif
// per-pass scaling of the lag (nf_body): known pass x3/4 (P2P widths), after the sweep x3/2
#ifndef SS_LAG_KNOWN_NUM
#define SS_LAG_KNOWN_NUM 3
#define SS_LAG_KNOWN_DEN 4
#endif
#ifndef SS_LAG_SWEEP_NUM
#define SS_LAG_SWEEP_NUM 3
#define SS_LAG_SWEEP_DEN 2
#endif

constexpr int kEarlySync = -3;  // vote_or_early: a peer proved the step sync before its sweep ended
constexpr int kEarlyChunks = 8;  // the early vote's ||g||^2 sweep reports its running sum this often

// order bits of one launch, decided once per block at kernel start
constexpr int kNormFirst = 1, kKnown = 2, kSafe = 4;

__device__ __forceinline__ void red_add_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed_sys(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Order predictor (adaptive mode): P(sync) per context of the last two agreed
// decisions, each an EWMA (weight 1/4) of the decisions that followed that
// context; pr[4] holds the context (0..3). A 2-bit history learns runs
// (context LL -> local, SS -> sync) as well as alternations, where a single
// EWMA would sit near 0.5 and pick the norm-first order for every local step.
// Every rank updates it from the same agreed words: all ranks pick the same order.
// Thread 0 of every block loads the predictor once at kernel start (five
// independent loads, then a select: no dependent load); the last block reuses
// that copy for the update at the end (nothing else writes the predictor
// during a launch), so the update costs two stores and no load latency.
struct PredCache {
    float p[4];
    int h;
};
__device__ __forceinline__ PredCache predictor_load(const float* pr) {
    const volatile float* v = pr;
    PredCache c;
    c.p[0] = v[0]; c.p[1] = v[1]; c.p[2] = v[2]; c.p[3] = v[3];
    c.h = static_cast<int>(v[4]) & 3;
    return c;
}
__device__ __forceinline__ float pick(const PredCache& c) {
    return c.h == 0 ? c.p[0] : c.h == 1 ? c.p[1] : c.h == 2 ? c.p[2] : c.p[3];
}
__device__ __forceinline__ void predictor_update(float* pr, const PredCache& c, int w) {
    const int s = w == SS_FLAG_SYNC ? 1 : 0;
    pr[c.h] = 0.75f * pick(c) + (s ? 0.25f : 0.0f);
    pr[4] = static_cast<float>(((c.h << 1) | s) & 3);
}

// bounded spin until *p >= want (gpu scope); sets the error word on timeout
__device__ void wait_count_gpu(const unsigned int* p, unsigned int want, const SymmArgs& s) {
    const uint64_t t0 = now_ns();
    while (*reinterpret_cast<const volatile unsigned int*>(p) < want) {
        if (now_ns() - t0 > s.timeout_ns) {
            atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
            return;
        }
        __nanosleep(32);
    }
    __threadfence();
}

// a peer met a NaN in an update tile of this step (known-sync pass)
__device__ bool poisoned(const SymmArgs& s, uint64_t seq) {
    bool p = false;
    for (int j = 0; j < s.world; ++j) p |= ld_acquire_sys(poison_slot(s, s.rank, j)) == seq;
    return p;
}

__device__ void post_poison(const SymmArgs& s, uint64_t seq) {
    fence_acq_rel_sys();
    for (int j = 0; j < s.world; ++j) st_relaxed_sys(poison_slot(s, j, s.rank), seq);
}

// end of a sync step on this rank: done tags to every peer, wait for all
__device__ void end_barrier(const SymmArgs& s, uint64_t seq) {
    fence_acq_rel_sys();
    for (int j = 0; j < s.world; ++j) st_relaxed_sys(done_slot(s, j, s.rank), seq);
    bool to = false;
    for (int j = 0; j < s.world && !to; ++j) wait_tag(done_slot(s, s.rank, j), seq, 0, s, &to);
    if (to) atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
}

// agreed word of step `seq` from the N seq-tagged votes in this rank's signal slots
__device__ int agreed_vote(const SymmArgs& s, uint64_t seq) {
    bool to = false;
    int w = 0;
    for (int j = 0; j < s.world && !to; ++j) {
        const uint64_t t = wait_tag(vote_slot(s, s.rank, seq, j), seq, 32, s, &to);
        const int wj = static_cast<int>(static_cast<uint32_t>(t));
        w = wj > w ? wj : w;
    }
    if (to) {
        atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
        return -1;
    }
    return w;
}

// Wait for the N final votes of step `seq` (returns their MAX, -1 on a
// timeout) or for an early sync tag from any rank, whichever comes first
// (returns kEarlySync). An early tag proves its rank's final vote is sync (or
// an error word), so the agreed word is >= SS_FLAG_SYNC: the mean may start.
__device__ int vote_or_early(const SymmArgs& s, uint64_t seq) {
    const uint64_t t0 = now_ns();
    for (;;) {
        int w = 0, have = 0;
        for (int j = 0; j < s.world; ++j) {
            const uint64_t t = ld_acquire_sys(vote_slot(s, s.rank, seq, j));
            if ((t >> 32) == seq) {
                ++have;
                const int wj = static_cast<int>(static_cast<uint32_t>(t));
                w = wj > w ? wj : w;
            }
        }
        if (have == s.world) return w;
        for (int j = 0; j < s.world; ++j)
            if (ld_acquire_sys(early_slot(s, s.rank, j)) == seq) return kEarlySync;
        if (now_ns() - t0 > s.timeout_ns) {
            atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
            return -1;
        }
        __nanosleep(64);
    }
}

// Known-sync pass: called by every thread of the block that just finished an
// update tile (its ||g||^2 partial is in tile_norm). The block finishing the
// last tile of this rank reduces the partials in tile order (deterministic),
// runs K2 and posts this rank's vote.
__device__ void known_tile_done(const Finish& f, const SymmArgs& s, const OverlapArgs& o, uint64_t seq, int N,
                                int64_t T, VBlk vb) {
    __shared__ bool s_last_tile;
    Workspace ws = ws_view(f.ws);
    if (threadIdx.x == 0) {
        __threadfence();
        s_last_tile = atomicAdd(ws.counter, 1u) == static_cast<unsigned int>(T - 1);
    }
    __syncthreads();
    if (!s_last_tile) return;
    __threadfence();
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < T; i += blockDim.x) v += __ldcg(o.tile_norm + i);
    v = block_sum(v);
    if (threadIdx.x == 0) {
        *ws.counter = 0u;
        // K2 advances step_count, which every block reads once at kernel start
        // to pick this launch's order: run it only after all of them have
        wait_count_gpu(o.started, static_cast<unsigned int>(vb.n), s);
        const int own = signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
        const uint64_t tagged = (seq << 32) | static_cast<uint32_t>(own);
        vote_fence();
        fence_acq_rel_sys();
        for (int j = 0; j < N; ++j) st_relaxed_sys(vote_slot(s, j, seq, s.rank), tagged);
        if (o.dbg) o.dbg[4 * o.dbg_cap + 1] = now_ns();
    }
}

// The decision of this step is sync before ||g||^2 is known: warmup (the
// observation about to be made is number <= warmup, signal.py:105-106) or
// delta == 0 (Delta >= 0 always). Same on every rank (same step count, delta).
__device__ __forceinline__ bool sync_known_ahead(const Finish& f) {
    const volatile ss_signal_state* st = f.st;
    return sync_known_ahead_core(st->step_count, st->warmup, f.delta, st->ewma_current);
}

// This launch's order, read by thread 0 of every block from state that only
// the last block of the PREVIOUS launch (predictor) or a K2 that waits for
// every block's arrival here (known pass) writes: all blocks agree. Only the
// known pass runs K2 before every block has arrived at the norm counter, so
// only a known snapshot counts itself in `started` (no 1-per-block atomic on
// other steps): K2 of the known pass waits for all of them, hence every block
// reads the state before K2 changes it and takes the known snapshot too.
// pc: thread 0's copy of the predictor (adaptive mode), for the update at the end.
__device__ int order_snapshot(const Finish& f, const OverlapArgs& o, PredCache* pc) {
    __shared__ int s_order;
    if (threadIdx.x == 0) {
        if (o.mode == 2) *pc = predictor_load(o.predictor);
        const bool known = (o.mode == 1 || o.mode == 2) && o.tile_norm != nullptr && sync_known_ahead(f);
        const bool nf = known || o.mode == 1 || o.mode == 3 || (o.mode == 2 && pick(*pc) >= o.threshold);
        s_order = (nf ? kNormFirst : 0) | (known ? kKnown : 0) | (o.mode == 3 ? kSafe : 0);
        if (known) {
            __threadfence();  // the state reads above complete before the arrival below
            atomicAdd(o.started, 1u);
        }
    }
    __syncthreads();
    return s_order;
}

template <bool MOM, bool NEST, int W>
__device__ __forceinline__ void nf_body(const SgdArgs& a, const Finish& f, const SymmArgs& s, const OverlapArgs& o,
                                     uint64_t seq, bool known, bool safe, VBlk vb, const PredCache& pc) {
    __shared__ unsigned long long s_ticket;
    __shared__ int s_vote;
    __shared__ bool s_last;
    __shared__ bool s_go;
    const int N = s.world;
    const int64_t T = o.n_tiles;
    // groups between a tile's update tickets and its mean ticket: o.lag (one
    // in-flight window) scaled per pass -- the pass after the ||g||^2 sweep
    // meets its updates already streaming and gains from a longer lag (x3/2:
    // -1.4 to -1.7 us per mixed step at N = 2 and 4); the known pass starts
    // its means with the first updates, and over P2P (N = 2) a shorter lag
    // (x3/4) gains 5-7 us per sync step, while over NVLS (N = 4) two same-box
    // A/Bs disagree in sign (+-6 us), so NVLS keeps the base lag
    // (profiles/r02_lag4/)
    const int lag = known ? (W == 0 ? o.lag : (o.lag - 2) * SS_LAG_KNOWN_NUM / SS_LAG_KNOWN_DEN + 2)
                          : (o.lag - 2) * SS_LAG_SWEEP_NUM / SS_LAG_SWEEP_DEN + 2;
    const int64_t groups = (T + N - 1) / N + lag;
    const unsigned long long total = static_cast<unsigned long long>(groups) * (N + 1);
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(o.epoch) + 1;
    const uint32_t target = static_cast<uint32_t>(N) * epoch;
    // known: the decision is sync whatever ||g||^2 turns out to be (warmup or
    // delta == 0, identical on every rank), so the mean tickets need no vote;
    // ||g||^2 then comes from the update tiles themselves (no separate sweep)
    // and the vote is still exchanged at the end, for the trace, the EWMA and
    // the error bits.
    // early: the exact early vote -- each block adds its ||g||^2 partial to a
    // running sum; once that lower bound proves the vote sync (upward jump,
    // sync_proven_early_core) the block posts an early sync tag to every rank
    // and the mean tickets start before the sweep ends. A NaN tile then
    // poisons its mean (as in the known pass): the final vote comes later.
    const bool early = o.early && !known && !safe;
    __shared__ bool s_early;
    if (threadIdx.x == 0) {
        s_vote = known ? SS_FLAG_SYNC : -2;
        s_early = false;
    }
    // ---- phase 1: ||g||^2 by the whole grid (full-speed sweep); the last block
    //      to arrive reduces the partials in a fixed order, runs K2 and posts the
    //      vote. Nobody waits here: blocks go straight on to the update tickets.
    if (!known) {
        Workspace ws = ws_view(f.ws);
        double bsum;
        if (early) {
            // the sweep in kEarlyChunks grid-strided chunks: after each one every
            // block adds what it summed to the running lower bound, which so grows
            // with the sweep instead of arriving all at once at its end
            double acc = 0.0, prev = 0.0;
            for (int c = 0; c < kEarlyChunks; ++c) {
                acc = norm_chunk<4>(a.g, a.n, a.head, vb, c, kEarlyChunks, acc);
                const double cum = block_sum(acc);
                if (threadIdx.x == 0) {
                    const double lower = atomicAdd(o.running, cum - prev) + (cum - prev);
                    prev = cum;
                    if (ld_relaxed_gpu(o.early_posted) != seq && sync_proven_early_core(f.st, lower, f.delta)) {
                        *reinterpret_cast<volatile uint64_t*>(o.early_posted) = seq;
                        fence_acq_rel_sys();
                        for (int j = 0; j < N; ++j) st_relaxed_sys(early_slot(s, j, s.rank), seq);
                        if (o.dbg) o.dbg[4 * o.dbg_cap + 3] = now_ns();
                    }
                }
            }
            bsum = prev;
        } else {
            bsum = block_sum(norm_pass<4>(a.g, a.n, a.head, vb));
        }
        if (threadIdx.x == 0) {
            ws.partials[vb.bid] = bsum;
            __threadfence();
            s_last = atomicAdd(ws.counter, 1u) == static_cast<unsigned int>(vb.n - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            double v = 0.0;
            for (int i = threadIdx.x; i < vb.n; i += blockDim.x) v += __ldcg(ws.partials + i);
            v = block_sum(v);
            if (threadIdx.x == 0) {
                *ws.counter = 0u;
                if (early) *o.running = 0.0;  // every block has added its partial
                const int own = signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
                const uint64_t tagged = (seq << 32) | static_cast<uint32_t>(own);
                vote_fence();
                fence_acq_rel_sys();
                for (int j = 0; j < N; ++j) st_relaxed_sys(vote_slot(s, j, seq, s.rank), tagged);
                if (o.dbg) o.dbg[4 * o.dbg_cap + 1] = now_ns();
            }
        }
    }
    __syncthreads();
    // ---- phase 2: tickets -- groups of N update tiles + 1 mean of an owned tile.
    //      The next ticket is fetched while this one is worked on (its atomic
    //      latency hides behind the tile); a block still takes its tickets in
    //      increasing order, so tickets only ever wait on earlier ones.
    unsigned long long nxt = 0;
    if (threadIdx.x == 0) nxt = atomicAdd(o.ticket, 1ull);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = nxt;
        __syncthreads();
        const unsigned long long k = s_ticket;
        __syncthreads();
        if (k >= total) break;
        if (threadIdx.x == 0) nxt = atomicAdd(o.ticket, 1ull);
        const bool rec = o.dbg != nullptr && static_cast<int64_t>(k) < o.dbg_cap && threadIdx.x == 0;
        uint64_t t_start = rec ? now_ns() : 0, t_ready = 0;
        int64_t rec_tile = -1;
        int kind = 0;
        {
            const unsigned long long k2 = k;
            const int64_t grp = static_cast<int64_t>(k2 / (N + 1));
            const int pos = static_cast<int>(k2 % (N + 1));
            if (pos < N) {
                // ---- update tile t (owner t % N), announced to the owner
                const int64_t t = grp * N + pos;
                if (t < T) {
                    const int64_t e0 = t * o.tile, e1 = e0 + o.tile < a.n ? e0 + o.tile : a.n;
                    if (safe) {
                        // NaN-safe order: no update before the agreed vote; an
                        // error bit on any rank (or a timeout) skips every update
                        if (threadIdx.x == 0 && s_vote == -2) s_vote = agreed_vote(s, seq);
                        __syncthreads();
                    }
                    if (safe && (s_vote & ~SS_FLAG_SYNC) != 0) {
                        // counted all the same: tile counts advance by N every norm-first step
                    } else if (!known) {
                        const double bad = sgd_block_range<MOM, NEST, 2, false, false, true>(a, e0, e1);
                        // the barrier orders the block's stores before the count below;
                        // a NaN in this tile poisons its mean if the early vote runs it
                        if (__syncthreads_or(bad != 0.0) && early && threadIdx.x == 0) post_poison(s, seq);
                    } else {
                        // block_sum's barriers also order the block's stores
                        const double ts = block_sum(sgd_block_range<MOM, NEST, 1, false, true>(a, e0, e1));
                        if (threadIdx.x == 0) {
                            o.tile_norm[t] = ts;
                            // a NaN in this tile: no owner may average anything from
                            // here on (the mean runs before the vote carries the error);
                            // the tag is released before this tile's count below
                            if (ts != ts) post_poison(s, seq);
                        }
                    }
                    // release at sys scope: the block's stores (ordered by the
                    // barrier) are visible to the owner before the count
                    if (threadIdx.x == 0) red_add_release_sys(o.cnt[t % N] + t, 1u);
                    if (known) known_tile_done(f, s, o, seq, N, T, vb);
                    rec_tile = t;
                }
            } else {
                // ---- mean of owned tile t: needs the agreed vote and all N updates
                const int64_t m = grp - lag;
                const int64_t t = m * N + s.rank;
                if (m >= 0 && t < T) {
                    if (threadIdx.x == 0) {
                        if (s_vote == -2 && !s_early) {
                            const int r = early ? vote_or_early(s, seq) : agreed_vote(s, seq);
                            if (r == kEarlySync) s_early = true;
                            else s_vote = r;
                        }
                        bool go = s_early || s_vote == SS_FLAG_SYNC;
                        if (go) {
                            const uint64_t t0 = now_ns();
                            while (static_cast<int32_t>(ld_acquire_sys_u32(o.cnt[s.rank] + t) - target) < 0) {
                                if (now_ns() - t0 > s.timeout_ns) {
                                    atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
                                    go = false;
                                    break;
                                }
                                __nanosleep(128);
                            }
                            // known pass: a NaN met by any rank before its count
                            // of this tile stops the mean here (acquired above)
                            if (go && (known || s_early) && poisoned(s, seq)) go = false;
                        }
                        s_go = go;
                    }
                    __syncthreads();
                    if (s_go) {
                        if (rec) t_ready = now_ns();
                        const int64_t e0 = t * o.tile, e1 = e0 + o.tile < a.n ? e0 + o.tile : a.n;
                        average_block_range<W>(s, e0, e1);
                        rec_tile = t;
                        kind = 1;
                    }
                }
            }
        }
        if (rec && rec_tile >= 0) {
            uint64_t* e = o.dbg + 4 * k;
            e[0] = (static_cast<uint64_t>(kind) << 48) | static_cast<uint64_t>(rec_tile);
            e[1] = t_start;
            e[2] = t_ready ? t_ready : t_start;
            e[3] = now_ns();
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(s.arrive, 1u) == static_cast<unsigned int>(vb.n - 1)) {
        const int w = (s_vote != -2 && !known) ? s_vote : agreed_vote(s, seq);
        if (o.dbg) o.dbg[4 * o.dbg_cap + 4] = now_ns();
        *f.word = w;
        if (s.agreed_ring && s.ring_cap > 0) s.agreed_ring[(seq - 1) % s.ring_cap] = w;
        if (o.mode == 2) predictor_update(o.predictor, pc, w);
        // known: the mean ran in any case; early: it may have run on an error step
        if (w == SS_FLAG_SYNC || known || (early && w > 0)) end_barrier(s, seq);
        if (o.dbg) o.dbg[4 * o.dbg_cap + 5] = now_ns();
        *o.ticket = 0ull;
        *o.epoch = epoch;
        *o.started = 0u;
        *s.arrive = 0u;
        *s.seq = static_cast<uint32_t>(seq);
    }
}

// update-first order: K13 over the whole buffer; the last block to arrive
// runs K2 and the vote exchange and broadcasts the agreed word to the other
// blocks of the grid (all co-resident: one wave), which wait for it instead
// of exiting. On sync every block then averages its part of this rank's
// shard (C2, 1/N in the epilogue) and the last one runs the end barrier --
// no second launch, no device-side launch.
template <bool MOM, bool NEST, int W>
__device__ __forceinline__ void uf_body(const SgdArgs& a, const Finish& f, const SymmArgs& s, const OverlapArgs& o,
                                     uint64_t seq, VBlk vb, const PredCache& pc) {
    __shared__ bool s_last;
    __shared__ int s_w;
    uint64_t* mark = o.dbg ? o.dbg + 4 * o.dbg_cap : nullptr;
    uint64_t* decided = reinterpret_cast<uint64_t*>(static_cast<char*>(f.ws) + 192);  // (seq << 32) | word
    const double acc = sgd_pass<MOM, NEST, true, (MOM ? 1 : 2)>(a, vb);
    Workspace ws = ws_view(f.ws);
    const double bsum = block_sum(acc);
    if (threadIdx.x == 0) {
        if (vb.n == 1) {
            s_last = true;  // one block (small P): no partials round trip
        } else {
            ws.partials[vb.bid] = bsum;
            // gpu scope suffices: the last block observes this counter, then
            // releases the vote at system scope (causality is transitive), so
            // peers reading after the vote see these stores
            __threadfence();
            s_last = atomicAdd(ws.counter, 1u) == static_cast<unsigned int>(vb.n - 1);
        }
    }
    __syncthreads();
    if (s_last) {
        double v = bsum;  // thread 0's value counts
        if (vb.n > 1) {
            __threadfence();
            v = 0.0;
            for (int i = threadIdx.x; i < vb.n; i += blockDim.x) v += __ldcg(ws.partials + i);
            v = block_sum(v);
        }
        if (threadIdx.x == 0) {
            *ws.counter = 0u;
            const int own = signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
            const uint64_t tagged = (seq << 32) | static_cast<uint32_t>(own);
            vote_fence();
            fence_acq_rel_sys();
            for (int j = 0; j < s.world; ++j) st_relaxed_sys(vote_slot(s, j, seq, s.rank), tagged);
            if (mark) mark[1] = now_ns();
            const int w = agreed_vote(s, seq);
            if (mark) mark[2] = now_ns();
            *f.word = w;
            if (s.agreed_ring && s.ring_cap > 0) s.agreed_ring[(seq - 1) % s.ring_cap] = w;
            st_release_gpu(decided, (seq << 32) | static_cast<uint32_t>(w));  // the waiting blocks first
            s_w = w;
            if (o.mode == 2) predictor_update(o.predictor, pc, w);
        }
    } else if (threadIdx.x == 0) {
        bool to = false;
        const uint64_t t = wait_tag_gpu(decided, seq, s.timeout_ns, &to, SS_DECIDED_SLEEP);
        if (to) atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
        s_w = to ? -1 : static_cast<int>(static_cast<uint32_t>(t));
    }
    __syncthreads();
    if (s_w != SS_FLAG_SYNC) {
        if (s_last && threadIdx.x == 0) *s.seq = static_cast<uint32_t>(seq);
        return;
    }
    average_shard<W>(s, vb);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(s.arrive, 1u) == static_cast<unsigned int>(vb.n - 1)) {
        end_barrier(s, seq);
        *s.arrive = 0u;
        *s.seq = static_cast<uint32_t>(seq);
    }
}

template <bool MOM, bool NEST, int W>
__device__ __forceinline__ void step_body(const SgdArgs& a, const Finish& f, const SymmArgs& s, const OverlapArgs& o,
                                          VBlk vb) {
    const uint64_t seq = static_cast<uint64_t>(*reinterpret_cast<volatile uint32_t*>(s.seq)) + 1;
    // the order of this step: identical on every rank (same decision history)
    PredCache pc{};
    const int order = order_snapshot(f, o, &pc);
    uint64_t* mark = o.dbg ? o.dbg + 4 * o.dbg_cap : nullptr;  // {start, vote posted, votes in, -, last arrival, end}
    if (mark && vb.bid == 0 && threadIdx.x == 0) mark[0] = now_ns();
    if (order & kNormFirst) {
        nf_body<MOM, NEST, W>(a, f, s, o, seq, (order & kKnown) != 0, (order & kSafe) != 0, vb, pc);
        return;
    }
    uf_body<MOM, NEST, W>(a, f, s, o, seq, vb, pc);
}

template <bool MOM, bool NEST, int W>
__global__ void __launch_bounds__(kThreads, 4) step_kernel(SgdArgs a, Finish f, SymmArgs s, OverlapArgs o) {
    pdl_wait();
    pdl_trigger();
    step_body<MOM, NEST, W>(a, f, s, o, hw_blk());
}

// ------------------------------------------- gradient aggregation, one launch
//
// _selsync_step with aggregation="grads" (strategies.py:395-399): the vote
// precedes the update, and on sync the update uses the MEAN gradient
// (runtime.py:259-273 does not store it). The flat gradient buffer lives in
// symmetric memory. ||g||^2 sweep + vote (as in the norm-first pass), then
// tickets: the mean of one tile this rank owns (NVLS / P2P, written back into
// every rank's gradient, then announced to every rank by a remote atomic
// add), followed `lag` groups later by N tile updates, each of which -- on a
// sync step -- waits for its tile's announcement. On a local step no ticket
// waits and the update uses the rank's own gradient.
template <bool MOM, bool NEST, int W>
__device__ __forceinline__ void ga_body(const SgdArgs& a, const Finish& f, const SymmArgs& s, const OverlapArgs& o,
                                        VBlk vb) {
    __shared__ unsigned long long s_ticket;
    __shared__ int s_vote;
    __shared__ bool s_last;
    const uint64_t seq = static_cast<uint64_t>(*reinterpret_cast<volatile uint32_t*>(s.seq)) + 1;
    const int N = s.world;
    const int64_t T = o.n_tiles;
    const int64_t groups = (T + N - 1) / N + o.lag;
    const unsigned long long total = static_cast<unsigned long long>(groups) * (N + 1);
    const uint32_t epoch = *reinterpret_cast<volatile uint32_t*>(o.epoch) + 1;  // sync steps so far + 1
    if (threadIdx.x == 0) s_vote = -2;
    {   // ---- ||g||^2 sweep; the last block runs K2 and posts the vote
        Workspace ws = ws_view(f.ws);
        const double bsum = block_sum(norm_pass<4>(a.g, a.n, a.head, vb));
        if (threadIdx.x == 0) {
            ws.partials[vb.bid] = bsum;
            __threadfence();
            s_last = atomicAdd(ws.counter, 1u) == static_cast<unsigned int>(vb.n - 1);
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            double v = 0.0;
            for (int i = threadIdx.x; i < vb.n; i += blockDim.x) v += __ldcg(ws.partials + i);
            v = block_sum(v);
            if (threadIdx.x == 0) {
                *ws.counter = 0u;
                const int own = signal_step_dev(f.st, v, f.delta, f.word, f.trace, f.cap);
                const uint64_t tagged = (seq << 32) | static_cast<uint32_t>(own);
                vote_fence();
                fence_acq_rel_sys();
                for (int j = 0; j < N; ++j) st_relaxed_sys(vote_slot(s, j, seq, s.rank), tagged);
            }
        }
    }
    __syncthreads();
    // every ticket needs the branch: the agreed vote (all ranks finished their
    // sweep -- the means overwrite the gradients the sweeps read, so there is
    // no early vote here)
    if (threadIdx.x == 0) s_vote = agreed_vote(s, seq);
    __syncthreads();
    const bool sync = s_vote == SS_FLAG_SYNC;
    // the vote precedes every update here: an error bit on any rank (or a
    // timeout) leaves w and m untouched on every rank (strategies.py:286 raises
    // before the deferred update of :395-399)
    const bool skip = (s_vote & ~SS_FLAG_SYNC) != 0;
    unsigned long long nxt = 0;  // next ticket fetched ahead, as in nf_body
    if (threadIdx.x == 0) nxt = atomicAdd(o.ticket, 1ull);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = nxt;
        __syncthreads();
        const unsigned long long k = s_ticket;
        __syncthreads();
        if (k >= total) break;
        if (threadIdx.x == 0) nxt = atomicAdd(o.ticket, 1ull);
        const int64_t grp = static_cast<int64_t>(k / (N + 1));
        const int pos = static_cast<int>(k % (N + 1));
        if (pos == 0) {
            // ---- mean of owned tile t = grp*N + rank, then announce it to every rank
            const int64_t t = grp * N + s.rank;
            if (sync && t < T) {
                const int64_t e0 = t * o.tile, e1 = e0 + o.tile < a.n ? e0 + o.tile : a.n;
                average_block_range<W>(s, e0, e1);
                __syncthreads();
                if (threadIdx.x == 0) {
                    fence_acq_rel_sys();
                    for (int j = 0; j < N; ++j) red_add_relaxed_sys(o.cnt[j] + t, 1u);
                }
            }
        } else {
            // ---- update tile t of group grp - lag (owner t % N), with the mean gradient on sync
            const int64_t t = (grp - o.lag) * N + (pos - 1);
            if (grp >= o.lag && t < T) {
                if (sync && threadIdx.x == 0) {
                    const uint64_t t0 = now_ns();
                    while (static_cast<int32_t>(ld_acquire_sys_u32(o.cnt[s.rank] + t) - epoch) < 0) {
                        if (now_ns() - t0 > s.timeout_ns) {
                            atomicExch(s.err, SS_SYMM_ERR_TIMEOUT);
                            break;
                        }
                        __nanosleep(128);
                    }
                }
                __syncthreads();
                const int64_t e0 = t * o.tile, e1 = e0 + o.tile < a.n ? e0 + o.tile : a.n;
                if (!skip) sgd_block_range<MOM, NEST, 2, true>(a, e0, e1);
            }
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(s.arrive, 1u) == static_cast<unsigned int>(vb.n - 1)) {
        *f.word = s_vote;
        if (s.agreed_ring && s.ring_cap > 0) s.agreed_ring[(seq - 1) % s.ring_cap] = s_vote;
        if (sync) {
            end_barrier(s, seq);  // no rank reuses its gradient buffer while a peer still reads it
            *o.epoch = epoch;
        }
        *o.ticket = 0ull;
        *s.arrive = 0u;
        *s.seq = static_cast<uint32_t>(seq);
    }
}

template <bool MOM, bool NEST, int W>
__global__ void __launch_bounds__(kThreads, 4) step_ga_kernel(SgdArgs a, Finish f, SymmArgs s, OverlapArgs o) {
    pdl_wait();
    pdl_trigger();
    ga_body<MOM, NEST, W>(a, f, s, o, hw_blk());
}

template <typename K>
int occupancy(K kernel, int threads) {
    int x = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, kernel, threads, 0) != cudaSuccess || x <= 0) x = 1;
    return x;
}

// SS_COOP=0 drops the cooperative attribute (A/B timing of the attribute only)
bool coop_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("SS_COOP");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// Grid of a one-launch step: one wave (#SMs x resident blocks, fewer for small
// P), capped by the group's max_blocks (ranks sharing one device split it).
int step_grid(int64_t vec_work, int per_thread, int resident, int max_blocks) {
    int grid = static_cast<int>(grid_for(vec_work, per_thread, resident));
    if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
    return grid;
}

// The blocks of a step kernel wait on each other (decision broadcast, tile
// tickets, the known pass's snapshot count), so the grid must be co-resident:
// a cooperative launch makes the driver place every block at once or fail the
// launch (cudaErrorCooperativeLaunchTooLarge -> SS_ERR_CONFIG) instead of
// letting a partly placed grid spin into the timeout. Capturable in CUDA graphs.
template <typename... P, typename... A>
int launch_coop(void (*kernel)(P...), int grid, void* stream, const char* what, A... args) {
    const cudaError_t e = launch_ex(kernel, grid, kThreads, static_cast<cudaStream_t>(stream), coop_enabled(), args...);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(e == cudaErrorCooperativeLaunchTooLarge ? SS_ERR_CONFIG : SS_ERR_CUDA,
                    "%s: %s (grid %d of %d threads: every block must be co-resident)", what,
                    cudaGetErrorString(e), grid, kThreads);
    }
    return check_launch(what);
}

template <bool MOM, bool NEST, int W>
int launch_step(const SgdArgs& a, Finish f, const SymmArgs& sa, OverlapArgs o, int max_blocks, void* stream) {
    static int res_step = 0;
    if (res_step == 0) res_step = occupancy(step_kernel<MOM, NEST, W>, kThreads);
    const int grid = step_grid((a.n - a.head) / 4 + 1, (MOM ? 1 : 2) * SS_STEP_PER_THREAD, res_step, max_blocks);
    f.total_blocks = grid;
    // norm-first pass: the in-flight window is ~grid tickets = grid / (N + 1)
    // groups; the mean of a tile is scheduled one window after its update
    // (SS_LAG_SCALE: A/B builds of another lag; 1/2, 1/4 and 0 measured slower)
    o.lag = static_cast<int>(grid / (sa.world + 1) * SS_LAG_SCALE) + 2;
    return launch_coop(step_kernel<MOM, NEST, W>, grid, stream, "ss_step_symm_f32", a, f, sa, o);
}

template <int W>
int dispatch_step(const SgdArgs& a, const Finish& f, const SymmArgs& sa, const OverlapArgs& o, bool mom,
                  bool nest, int max_blocks, void* stream) {
    if (!mom) return launch_step<false, false, W>(a, f, sa, o, max_blocks, stream);
    if (nest) return launch_step<true, true, W>(a, f, sa, o, max_blocks, stream);
    return launch_step<true, false, W>(a, f, sa, o, max_blocks, stream);
}


template <bool MOM, bool NEST, int W>
int launch_step_ga(const SgdArgs& a, Finish f, const SymmArgs& sa, OverlapArgs o, int max_blocks, void* stream) {
    static int res = 0;
    if (res == 0) res = occupancy(step_ga_kernel<MOM, NEST, W>, kThreads);
    const int grid = step_grid((a.n - a.head) / 4 + 1, MOM ? 1 : 2, res, max_blocks);
    f.total_blocks = grid;
    o.lag = grid / (sa.world + 1) + 2;
    return launch_coop(step_ga_kernel<MOM, NEST, W>, grid, stream, "ss_step_symm_ga_f32", a, f, sa, o);
}

template <int W>
int dispatch_step_ga(const SgdArgs& a, const Finish& f, const SymmArgs& sa, const OverlapArgs& o, bool mom,
                     bool nest, int max_blocks, void* stream) {
    if (!mom) return launch_step_ga<false, false, W>(a, f, sa, o, max_blocks, stream);
    if (nest) return launch_step_ga<true, true, W>(a, f, sa, o, max_blocks, stream);
    return launch_step_ga<true, false, W>(a, f, sa, o, max_blocks, stream);
}

}  // namespace

namespace {

// Argument blocks of one rank's one-launch step (both aggregation modes),
// validated. The host-launch entry points and the colocated plan share it.
struct RankArgs {
    SgdArgs a;
    Finish f;
    SymmArgs s;
    OverlapArgs o;
};

int build_rank_args(bool ga, float* w, float* g, float* m, int64_t n, float lr, float momentum, float dampening,
                    float weight_decay, int32_t nesterov, int32_t first_step, ss_signal_state* st, double delta,
                    int32_t* word, ss_trace_row* trace, int32_t cap, const ss_symm_group* grp, void* ws,
                    RankArgs* out) {
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
    if (grp->max_blocks < 0) return fail(SS_ERR_CONFIG, "max_blocks must be >= 0, got %d", grp->max_blocks);
    OverlapArgs o{};
    o.dbg = grp->debug_events;
    o.dbg_cap = grp->debug_events ? grp->debug_cap : 0;
    o.mode = ga ? 0 : (grp->order_mode & SS_ORDER_MODE_MASK);
    o.early = (!ga && (grp->order_mode & SS_ORDER_EARLY_VOTE)) ? 1 : 0;
    o.running = reinterpret_cast<double*>(static_cast<char*>(ws) + 160);
    o.early_posted = reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + 176);
    o.threshold = grp->order_threshold;
    o.started = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + 224);
    o.ticket = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 128);
    const bool tiled = ga || o.mode != 0;
    if (ga) {
        if (grp->bufs[grp->rank] != g) return fail(SS_ERR_CONFIG, "g must be this rank's symmetric buffer");
        if (a.head != 0) return fail(SS_ERR_CONFIG, "gradient aggregation needs 16-byte aligned w, g, m");
        if (!grp->epoch || grp->tile_elems <= 0 || (grp->tile_elems & 3))
            return fail(SS_ERR_CONFIG, "gradient aggregation needs epoch and a tile size (multiple of 4)");
    } else {
        if (grp->bufs[grp->rank] != w) return fail(SS_ERR_CONFIG, "w must be this rank's symmetric buffer");
        if ((grp->order_mode & ~(SS_ORDER_MODE_MASK | SS_ORDER_EARLY_VOTE)) != 0 || o.mode > 3)
            return fail(SS_ERR_CONFIG, "order_mode must be 0, 1, 2 or 3 (| SS_ORDER_EARLY_VOTE), got %d",
                        grp->order_mode);
        if (o.mode != 0) {
            if (a.head != 0) return fail(SS_ERR_CONFIG, "norm-first order needs 16-byte aligned w, g, m");
            if (!grp->epoch || !grp->predictor || grp->tile_elems <= 0 || (grp->tile_elems & 3))
                return fail(SS_ERR_CONFIG, "norm-first order needs epoch, predictor and a tile size (multiple of 4)");
        }
    }
    if (tiled) {
        const int64_t tiles = (n + grp->tile_elems - 1) / grp->tile_elems;
        if (tiles > grp->n_tiles) return fail(SS_ERR_CONFIG, "tile counters hold %lld tiles, need %lld",
                                             (long long)grp->n_tiles, (long long)tiles);
        for (int r = 0; r < kMaxRanks; ++r) {
            if (r < grp->world && !grp->tile_cnt[r]) return fail(SS_ERR_CONFIG, "null tile counters for rank %d", r);
            o.cnt[r] = r < grp->world ? grp->tile_cnt[r] : nullptr;
        }
        o.epoch = grp->epoch;
        o.predictor = grp->predictor;
        o.tile = grp->tile_elems;
        o.n_tiles = tiles;
        if (!ga) o.tile_norm = grp->tile_norm;
    }
    out->a = a;
    out->f = Finish{ws, 0, 0, nullptr, st, delta, word, trace, cap};
    out->s = sa;
    out->o = o;
    return SS_OK;
}

// ------------------------------------------------ colocated ranks, one launch
//
// Ranks that share ONE device must not run as separate launches that wait on
// one another (nothing guarantees that they run at the same time). Their
// grids are therefore one cooperative launch: blocks [r*G, (r+1)*G) are rank
// r's grid of G blocks, each running exactly the code of the per-rank launch
// over its rank's argument block (kept in device memory, copied to shared
// memory per block) with its slice index as the block index.

__device__ __forceinline__ const RankArgs& load_rank_args(const RankArgs* __restrict__ args, int rank, float lr,
                                                          int first) {
    __shared__ __align__(16) RankArgs s_ra;
    static_assert(sizeof(RankArgs) % 16 == 0, "RankArgs copies in 16-byte vectors");
    const uint4* src = reinterpret_cast<const uint4*>(args + rank);
    uint4* dst = reinterpret_cast<uint4*>(&s_ra);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(RankArgs) / 16); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        s_ra.a.lr = lr;
        s_ra.a.first = first;
    }
    __syncthreads();
    return s_ra;
}

template <bool MOM, bool NEST, int W>
__global__ void __launch_bounds__(kThreads, 4) step_kernel_colo(const RankArgs* __restrict__ args, int per_rank,
                                                                float lr, int first) {
    pdl_wait();
    pdl_trigger();
    const int rank = static_cast<int>(blockIdx.x) / per_rank;
    const RankArgs& ra = load_rank_args(args, rank, lr, first);
    step_body<MOM, NEST, W>(ra.a, ra.f, ra.s, ra.o, VBlk{static_cast<int>(blockIdx.x) % per_rank, per_rank});
}

template <bool MOM, bool NEST, int W>
__global__ void __launch_bounds__(kThreads, 4) step_ga_kernel_colo(const RankArgs* __restrict__ args, int per_rank,
                                                                   float lr, int first) {
    pdl_wait();
    pdl_trigger();
    const int rank = static_cast<int>(blockIdx.x) / per_rank;
    const RankArgs& ra = load_rank_args(args, rank, lr, first);
    ga_body<MOM, NEST, W>(ra.a, ra.f, ra.s, ra.o, VBlk{static_cast<int>(blockIdx.x) % per_rank, per_rank});
}

template <bool MOM, bool NEST, int W>
void* colo_kernel(bool ga) {
    return ga ? reinterpret_cast<void*>(step_ga_kernel_colo<MOM, NEST, W>)
              : reinterpret_cast<void*>(step_kernel_colo<MOM, NEST, W>);
}

template <int W>
void* colo_kernel_for(bool ga, bool mom, bool nest) {
    if (!mom) return colo_kernel<false, false, W>(ga);
    return nest ? colo_kernel<true, true, W>(ga) : colo_kernel<true, false, W>(ga);
}

void* colo_kernel_any(int ranks, bool ga, bool mom, bool nest) {
    switch (ranks) {
        case 1: return colo_kernel_for<1>(ga, mom, nest);
        case 2: return colo_kernel_for<2>(ga, mom, nest);
        case 4: return colo_kernel_for<4>(ga, mom, nest);
        case 8: return colo_kernel_for<8>(ga, mom, nest);
        default: return nullptr;
    }
}

}  // namespace

extern "C" int ss_step_symm_f32(float* w, const float* g, float* m, int64_t n, float lr, float momentum,
                                float dampening, float weight_decay, int32_t nesterov, int32_t first_step,
                                ss_signal_state* st, double delta, int32_t* word, ss_trace_row* trace,
                                int32_t cap, const ss_symm_group* grp, void* ws, void* stream) {
    RankArgs r;
    const int rc = build_rank_args(false, w, const_cast<float*>(g), m, n, lr, momentum, dampening, weight_decay,
                                   nesterov, first_step, st, delta, word, trace, cap, grp, ws, &r);
    if (rc) return rc;
    const bool mom = momentum != 0.0f, nest = nesterov != 0;
    const int mb = grp->max_blocks;
    switch (symm_width(r.s)) {
        case 0: return dispatch_step<0>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 1: return dispatch_step<1>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);  // single rank (profiling)
        case 2: return dispatch_step<2>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 4: return dispatch_step<4>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 8: return dispatch_step<8>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        default:
            return fail(SS_ERR_CONFIG, "one-launch step: world %d needs multicast (P2P widths 1, 2, 4, 8)", r.s.world);
    }
}

extern "C" int ss_step_symm_ga_f32(float* w, float* g, float* m, int64_t n, float lr, float momentum,
                                   float dampening, float weight_decay, int32_t nesterov, int32_t first_step,
                                   ss_signal_state* st, double delta, int32_t* word, ss_trace_row* trace,
                                   int32_t cap, const ss_symm_group* grp, void* ws, void* stream) {
    RankArgs r;
    const int rc = build_rank_args(true, w, g, m, n, lr, momentum, dampening, weight_decay, nesterov, first_step,
                                   st, delta, word, trace, cap, grp, ws, &r);
    if (rc) return rc;
    const bool mom = momentum != 0.0f, nest = nesterov != 0;
    const int mb = grp->max_blocks;
    switch (symm_width(r.s)) {
        case 0: return dispatch_step_ga<0>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 1: return dispatch_step_ga<1>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 2: return dispatch_step_ga<2>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 4: return dispatch_step_ga<4>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        case 8: return dispatch_step_ga<8>(r.a, r.f, r.s, r.o, mom, nest, mb, stream);
        default:
            return fail(SS_ERR_CONFIG, "gradient aggregation: world %d needs multicast (P2P widths 1, 2, 4, 8)",
                        r.s.world);
    }
}

extern "C" int ss_colocated_args_bytes(int32_t ranks, int64_t* bytes) {
    if (!bytes) return fail(SS_ERR_CONFIG, "null output");
    if (ranks != 1 && ranks != 2 && ranks != 4 && ranks != 8)
        return fail(SS_ERR_CONFIG, "colocated ranks: 1, 2, 4 or 8 (the P2P widths of the step kernel), got %d", ranks);
    *bytes = static_cast<int64_t>(ranks) * static_cast<int64_t>(sizeof(RankArgs));
    return SS_OK;
}

extern "C" int ss_colocated_prepare_f32(const ss_rank_step* rs, int32_t ranks, int32_t grads,
                                        int32_t max_blocks_per_rank, ss_colocated_plan* plan, void* stream) {
    int64_t bytes = 0;
    int rc = ss_colocated_args_bytes(ranks, &bytes);
    if (rc) return rc;
    if (!rs || !plan || !plan->args_dev) return fail(SS_ERR_CONFIG, "null rank table / plan / plan->args_dev");
    if (max_blocks_per_rank < 0) return fail(SS_ERR_CONFIG, "max_blocks_per_rank must be >= 0");
    const bool ga = grads != 0;
    const bool mom = rs[0].momentum != 0.0f, nest = rs[0].nesterov != 0;
    RankArgs host[SS_SYMM_MAX_RANKS];
    for (int r = 0; r < ranks; ++r) {
        const ss_rank_step& x = rs[r];
        if (!x.group) return fail(SS_ERR_CONFIG, "rank %d: null group", r);
        if (x.group->world != ranks || x.group->rank != r)
            return fail(SS_ERR_CONFIG, "rank %d: group says rank %d of %d", r, x.group->rank, x.group->world);
        if (x.group->mc) return fail(SS_ERR_CONFIG, "colocated ranks have no multicast address");
        if (x.n != rs[0].n || (x.momentum != 0.0f) != mom || (x.nesterov != 0) != nest)
            return fail(SS_ERR_CONFIG, "rank %d: every colocated rank needs the same size and update kind", r);
        rc = build_rank_args(ga, x.w_dev, x.g_dev, x.m_dev, x.n, 0.0f, x.momentum, x.dampening, x.weight_decay,
                             x.nesterov, 0, x.st_dev, x.delta, x.word_dev, x.trace_dev, x.trace_cap, x.group, x.ws_dev,
                             &host[r]);
        if (rc) {
            char msg[384];
            snprintf(msg, sizeof(msg), "%s", ss_last_error());
            return fail(rc, "rank %d: %s", r, msg);
        }
    }
    // one cooperative launch of ranks x G blocks: G = this rank's one-wave grid,
    // capped so that all ranks' grids are co-resident together
    void* kern = colo_kernel_any(ranks, ga, mom, nest);
    int res = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, kern, kThreads, 0) != cudaSuccess || res <= 0)
        return check_launch("ss_colocated_prepare_f32 (occupancy)");
    const int cap = ss_internal::sm_count() * res / ranks;
    if (cap < 1) return fail(SS_ERR_CONFIG, "%d colocated grids do not fit on this device", ranks);
    int per_rank = static_cast<int>(grid_for((host[0].a.n - host[0].a.head) / 4 + 1, mom ? 1 : 2, res));
    if (per_rank > cap) per_rank = cap;
    if (max_blocks_per_rank > 0 && per_rank > max_blocks_per_rank) per_rank = max_blocks_per_rank;
    for (int r = 0; r < ranks; ++r) {
        host[r].f.total_blocks = per_rank;
        host[r].o.lag = per_rank / (ranks + 1) + 2;
    }
    if (cudaMemcpyAsync(plan->args_dev, host, static_cast<size_t>(bytes), cudaMemcpyHostToDevice,
                        static_cast<cudaStream_t>(stream)) != cudaSuccess ||
        cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return check_launch("ss_colocated_prepare_f32 (argument copy)");
    plan->ranks = ranks;
    plan->blocks_per_rank = per_rank;
    plan->grads = ga ? 1 : 0;
    plan->flags = (mom ? 1 : 0) | (nest ? 2 : 0);
    return SS_OK;
}

extern "C" int ss_colocated_step_f32(const ss_colocated_plan* plan, float lr, int32_t first_step, void* stream) {
    if (!plan || !plan->args_dev || plan->blocks_per_rank < 1) return fail(SS_ERR_CONFIG, "plan not prepared");
    if (!(lr >= 0.0f)) return fail(SS_ERR_CONFIG, "learning rate must be non-negative, got %g", (double)lr);
    const bool ga = plan->grads != 0, mom = plan->flags & 1, nest = (plan->flags & 2) != 0;
    void* kern = colo_kernel_any(plan->ranks, ga, mom, nest);
    if (!kern) return fail(SS_ERR_CONFIG, "bad plan (ranks %d)", plan->ranks);
    const RankArgs* args = static_cast<const RankArgs*>(plan->args_dev);
    int per_rank = plan->blocks_per_rank;
    int first = first_step ? 1 : 0;
    void* params[] = {&args, &per_rank, &lr, &first};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(plan->ranks * per_rank));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelExC(&cfg, kern, params);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(e == cudaErrorCooperativeLaunchTooLarge ? SS_ERR_CONFIG : SS_ERR_CUDA,
                    "ss_colocated_step_f32: %s (%d ranks x %d blocks)", cudaGetErrorString(e), plan->ranks, per_rank);
    }
    return check_launch("ss_colocated_step_f32");
}

// ------------------------------------------------ prepared per-rank step
//
// ss_step_plan_init validates a rank's step once (what ss_update_norm_signal_f32
// / ss_step_symm_f32 / ss_step_symm_ga_f32 check on every call), picks the
// kernel and keeps the argument blocks; ss_step_plan_launch patches the
// gradient, lr and first-step flag and launches. At small P the per-step host
// path is the step's cost, so the launch is one short call.

namespace {

constexpr uint32_t kPlanMagic = 0x53535031u;  // "SSP1"

struct PlanImpl {
    uint32_t magic;
    int32_t kind;        // 0: K13+K2 (one rank, no group), 1: one-launch step, 2: its GA form
    int32_t resident;    // blocks per SM of the kernel
    int32_t per_thread;  // float4 vectors per thread and stream the grid is sized for
    int32_t max_blocks;
    int32_t world;
    void* kernel;
    RankArgs r;
};
static_assert(sizeof(PlanImpl) <= sizeof(ss_step_plan), "ss_step_plan too small for the argument blocks");

template <bool MOM, bool NEST>
void* step_kernel_for_width(int width, bool ga) {
    switch (width) {
        case 0: return ga ? reinterpret_cast<void*>(step_ga_kernel<MOM, NEST, 0>) : reinterpret_cast<void*>(step_kernel<MOM, NEST, 0>);
        case 1: return ga ? reinterpret_cast<void*>(step_ga_kernel<MOM, NEST, 1>) : reinterpret_cast<void*>(step_kernel<MOM, NEST, 1>);
        case 2: return ga ? reinterpret_cast<void*>(step_ga_kernel<MOM, NEST, 2>) : reinterpret_cast<void*>(step_kernel<MOM, NEST, 2>);
        case 4: return ga ? reinterpret_cast<void*>(step_ga_kernel<MOM, NEST, 4>) : reinterpret_cast<void*>(step_kernel<MOM, NEST, 4>);
        case 8: return ga ? reinterpret_cast<void*>(step_ga_kernel<MOM, NEST, 8>) : reinterpret_cast<void*>(step_kernel<MOM, NEST, 8>);
        default: return nullptr;
    }
}

void* step_kernel_any(int width, bool ga, bool mom, bool nest) {
    if (!mom) return step_kernel_for_width<false, false>(width, ga);
    return nest ? step_kernel_for_width<true, true>(width, ga) : step_kernel_for_width<true, false>(width, ga);
}

}  // namespace

extern "C" int ss_step_plan_init(ss_step_plan* plan, const ss_rank_step* x, int32_t grads) {
    if (!plan || !x) return fail(SS_ERR_CONFIG, "null plan or rank descriptor");
    std::memset(plan, 0, sizeof(*plan));
    PlanImpl p{};
    const bool ga = grads != 0, mom = x->momentum != 0.0f, nest = x->nesterov != 0;
    int rc;
    if (!x->group) {
        // one rank without a group: K13+K2 (ss_update_norm_signal_f32)
        if (ga) return fail(SS_ERR_CONFIG, "gradient aggregation needs a symmetric group");
        rc = make_sgd_args(&p.r.a, x->w_dev, x->g_dev, x->m_dev, x->n, 0.0f, x->momentum, x->dampening,
                           x->weight_decay, x->nesterov, 0, nullptr, 1.0f);
        if (rc) return rc;
        if (!x->st_dev || !x->ws_dev) return fail(SS_ERR_CONFIG, "null state/workspace");
        rc = check_delta_impl(x->delta);
        if (rc) return rc;
        rc = check_trace(x->trace_dev, x->trace_cap);
        if (rc) return rc;
        p.r.f = Finish{x->ws_dev, 0, 0, nullptr, x->st_dev, x->delta, x->word_dev, x->trace_dev, x->trace_cap};
        p.kind = 0;
        p.kernel = ss_internal::k13_kernel(mom, nest, &p.per_thread);
        p.world = 1;
    } else {
        rc = build_rank_args(ga, x->w_dev, x->g_dev, x->m_dev, x->n, 0.0f, x->momentum, x->dampening,
                             x->weight_decay, x->nesterov, 0, x->st_dev, x->delta, x->word_dev, x->trace_dev,
                             x->trace_cap, x->group, x->ws_dev, &p.r);
        if (rc) return rc;
        const int width = symm_width(p.r.s);
        p.kernel = step_kernel_any(width, ga, mom, nest);
        if (!p.kernel)
            return fail(SS_ERR_CONFIG, "one-launch step: world %d needs multicast (P2P widths 1, 2, 4, 8)",
                        p.r.s.world);
        p.kind = ga ? 2 : 1;
        p.per_thread = ga ? (mom ? 1 : 2) : (mom ? 1 : 2) * SS_STEP_PER_THREAD;
        p.max_blocks = x->group->max_blocks;
        p.world = x->group->world;
    }
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.resident, p.kernel, kThreads, 0) != cudaSuccess ||
        p.resident <= 0)
        return check_launch("ss_step_plan_init (occupancy)");
    p.magic = kPlanMagic;
    std::memcpy(plan, &p, sizeof(p));
    return SS_OK;
}

extern "C" int ss_step_plan_launch(const ss_step_plan* plan, const float* g, float lr, int32_t first_step,
                                   void* stream) {
    if (!plan) return fail(SS_ERR_CONFIG, "step plan not initialised");
    PlanImpl pl;  // a copy: the caller's storage is plain words (no aliasing through it)
    std::memcpy(&pl, plan, sizeof(pl));
    const PlanImpl* p = &pl;
    if (p->magic != kPlanMagic) return fail(SS_ERR_CONFIG, "step plan not initialised");
    if (!(lr >= 0.0f)) return fail(SS_ERR_CONFIG, "learning rate must be non-negative, got %g", (double)lr);
    RankArgs& r = pl.r;
    const int64_t n = r.a.n;
    if (n > 0 && !g) return fail(SS_ERR_CONFIG, "null gradient pointer");
    if (p->kind == 2 && g != r.a.g) return fail(SS_ERR_CONFIG, "g must be this rank's symmetric buffer");
    r.a.g = g;
    r.a.lr = lr;
    r.a.first = first_step ? 1 : 0;
    r.a.head = n ? common_head(n, g, r.a.w, r.a.m) : 0;
    if (p->kind == 1 && r.o.mode != 0 && r.a.head != 0)
        return fail(SS_ERR_CONFIG, "norm-first order needs 16-byte aligned w, g, m");
    const int64_t work = (n - r.a.head) / 4 + 1;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (p->kind == 0) {
        const int grid = static_cast<int>(grid_for(work, p->per_thread, p->resident));
        r.f.total_blocks = grid;
        void* params[] = {&r.a, &r.f};
        (void)launch_ex_c(p->kernel, grid, kThreads, s, false, params);
        return check_launch("ss_step_plan_launch");
    }
    const int grid = step_grid(work, p->per_thread, p->resident, p->max_blocks);
    r.f.total_blocks = grid;
    r.o.lag = p->kind == 1 ? static_cast<int>(grid / (p->world + 1) * SS_LAG_SCALE) + 2 : grid / (p->world + 1) + 2;
    void* params[] = {&r.a, &r.f, &r.s, &r.o};
    const cudaError_t e = launch_ex_c(p->kernel, grid, kThreads, s, coop_enabled(), params);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(e == cudaErrorCooperativeLaunchTooLarge ? SS_ERR_CONFIG : SS_ERR_CUDA,
                    "ss_step_plan_launch: %s (grid %d of %d threads: every block must be co-resident)",
                    cudaGetErrorString(e), grid, kThreads);
    }
    return check_launch("ss_step_plan_launch");
}
