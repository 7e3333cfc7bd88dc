/*
 * selsync_b200.h -- C-ABI of the B200-native SelSync hot path.
 *
 * The reference (arXiv 2307.07950's desk-scale re-implementation,
 * /root/reference/pkg/src/selsync) has no FFI: its hot path is Python/numpy
 * behind the functions cited on each entry point below. This header is the
 * boundary a binding (ctypes / cffi / pybind) attaches to; see INTEGRATION.md.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / CUDA types in signatures
 *     (streams travel as `void*` = cudaStream_t, 0 = legacy default stream);
 *   - every function returns an int status: SS_OK or SS_ERR_*; the message of
 *     the last failure on the calling thread is ss_last_error();
 *   - "dev" arguments are device pointers (HBM), "host" arguments live in host
 *     memory; device kernels are asynchronous on the given stream;
 *   - a workspace (ss_workspace_bytes) is owned by one stream at a time;
 *   - the norm, update and step kernels are launched with programmatic stream
 *     serialization (programmatic dependent launch): their blocks may be
 *     placed while the previous kernel in the stream drains, and each waits
 *     (griddepcontrol.wait) for that kernel to complete before it touches
 *     memory, so stream order is unchanged for every caller. They also
 *     trigger their own dependents at entry. SS_PDL=0 in the environment
 *     launches them without the attribute.
 *
 * Build: nvcc -gencode arch=compute_100a,code=sm_100a (see __graft_entry__.py).
 */
#ifndef SELSYNC_B200_H
#define SELSYNC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 1

#if defined(__GNUC__)
#define SS_API __attribute__((visibility("default")))
#else
#define SS_API
#endif

/* status codes; the Python shim maps them onto selsync's exception types
   (errors.py:4-17): CONFIG -> ConfigError, SIGNAL -> SignalError */
#define SS_OK 0
#define SS_ERR_CONFIG 1
#define SS_ERR_SIGNAL 2
#define SS_ERR_CUDA 3

/* bits of the per-rank int32 flag word written by the signal step. Word
   values are 0/1 unless an error bit is set, so an allreduce-MAX over ranks
   is the N-bit OR of wire.py:139-151 / runtime.py:319-333, and any rank's
   error (>= 2) reaches every rank in the same collective. */
#define SS_FLAG_SYNC 1    /* own vote: decide() == "sync" (signal.py:101-107) */
#define SS_FLAG_ERR_NAN 2 /* observed NaN (signal.py:67-68); state unchanged */
#define SS_FLAG_ERR_NEG 4 /* observed x < 0 (signal.py:69-70); state unchanged */

/* GradSignalState (signal.py:41-61) as a 64-byte POD that lives in HBM for
   the device path or in host memory for the scalar API. */
typedef struct ss_signal_state {
    double smoothing;      /* lambda in (0, 1] */
    double ewma_current;
    double ewma_previous;
    double max_delta_seen;
    double last_delta;     /* relative_change after the last observe; NaN if step_count < 2 */
    double last_norm_sq;   /* last observed ||g||^2 */
    int64_t step_count;
    int32_t warmup;        /* >= 1; the "EWMA window" of the paper */
    int32_t error;         /* sticky SS_FLAG_ERR_* bits of rejected observations */
} ss_signal_state;

/* one decision-trace row (MetricsRecord columns grad_norm_sq, ewma, delta_g,
   decision; metrics.py:23-48), written into a device ring by the signal step */
typedef struct ss_trace_row {
    double grad_norm_sq;
    double ewma;
    double delta_g;        /* NaN where the reference records None (strategies.py:287) */
    int32_t step;          /* 0-based observation index of this worker */
    int32_t word;          /* SS_FLAG_* bits: own vote | errors */
} ss_trace_row;

SS_API int ss_abi_version(void);
SS_API const char* ss_last_error(void);
SS_API int ss_signal_state_size(void);
SS_API int ss_trace_row_size(void);

/* ---------------- host scalar API (no GPU needed) ---------------- */

/* default_smoothing, signal.py:20-29 */
SS_API int ss_default_smoothing(int32_t n_workers, double* out_host);
/* DeltaThreshold validation, signal.py:32-38 */
SS_API int ss_check_delta(double delta);
/* GradSignalState(smoothing, warmup) + __post_init__, signal.py:41-61 */
SS_API int ss_signal_init(ss_signal_state* st_host, double smoothing, int32_t warmup);
/* observe, signal.py:64-83; st unchanged on error */
SS_API int ss_signal_observe(ss_signal_state* st_host, double grad_norm_sq);
/* relative_change, signal.py:86-98 */
SS_API int ss_relative_change(const ss_signal_state* st_host, double* out_host);
/* decide, signal.py:101-107: *sync_out = 1 for "sync", 0 for "local" */
SS_API int ss_decide(const ss_signal_state* st_host, double delta, int32_t* sync_out_host);
/* *known_out = 1 when the NEXT decide (after one more observe of any finite
   ||g||^2 >= 0) is "sync" whatever that norm is: a warmup step or delta == 0.
   The one-launch step uses the same predicate on the device (known-sync pass).
   No reference counterpart: it restates signal.py:101-107 one step ahead. */
SS_API int ss_sync_known_ahead(const ss_signal_state* st_host, double delta, int32_t* known_out_host);

/* *proven_out_host = 1 when observing ANY total >= lower next (lower: a
   partial sum of the non-negative squares whose total is ||g||^2) is proven
   to vote "sync" on the upward side (new EWMA >= previous): the exact early
   vote of the norm-first step, which lets the mean start before the ||g||^2
   sweep ends. Sound, not complete (downward jumps are never proven early).
   No reference counterpart: it restates signal.py:64-107 for an interval. */
SS_API int ss_sync_proven_early(const ss_signal_state* st_host, double lower, double delta,
                                int32_t* proven_out_host);

/* ---------------- device hot path (sm_100a) ---------------- */

/* bytes of scratch (block partials + arrival counter) any kernel below needs;
   the memory must be zeroed once (ss_workspace_reset) and is then self-resetting */
SS_API int ss_workspace_bytes(int64_t* bytes_host);
SS_API int ss_workspace_reset(void* ws_dev, void* stream);

/* K1: ||g||^2 of one flat fp32 buffer in fp64, one launch, deterministic
   two-pass finish (last-arriving block reduces the block partials in a fixed
   order). Replaces float(grad @ grad), strategies.py:285. */
SS_API int ss_norm_sq_f32(const float* g_dev, int64_t n, double* out_dev, void* ws_dev, void* stream);

/* K1 over a list of tensors (pointer table, one logical launch per <= 256
   tensors; the model's p.grad tensors need not be contiguous). ptrs/sizes are
   HOST arrays of device pointers / element counts. out_dev and/or st_dev may
   be NULL; with st_dev the signal step (K2) runs in the finishing block. */
SS_API int ss_norm_sq_multi_f32(const float* const* ptrs_host, const int64_t* sizes_host, int32_t count,
                         double* out_dev, ss_signal_state* st_dev, double delta,
                         int32_t* word_dev, ss_trace_row* trace_dev, int32_t trace_cap,
                         void* ws_dev, void* stream);

/* K2 alone: observe + relative_change + decide on the device-resident state
   for a device-resident ||g||^2 (_grad_and_signal strategies.py:283-288 +
   decide :384). Writes the flag word and, if trace_dev != NULL, the row
   trace_dev[step % trace_cap]. One thread. */
SS_API int ss_signal_step(ss_signal_state* st_dev, const double* norm_sq_dev, double delta,
                   int32_t* word_dev, ss_trace_row* trace_dev, int32_t trace_cap, void* stream);

/* K1+K2 in one launch over a flat buffer (prescale / grads-aggregation order) */
SS_API int ss_norm_signal_f32(const float* g_dev, int64_t n, ss_signal_state* st_dev, double delta,
                       int32_t* word_dev, ss_trace_row* trace_dev, int32_t trace_cap,
                       void* ws_dev, void* stream);

/* K3: fused SGD (+momentum, +weight decay, optional Nesterov) in place:
     d = g + wd*w; m = first ? d : mu*m + (1-dampening)*d; d = nesterov ? d + mu*m : m;
     w = (w - lr*d) * s,  s = sync_scale if (sync_word_dev && *sync_word_dev & SS_FLAG_SYNC) else 1
   When *sync_word_dev carries an error bit (>= 2: some rank observed a NaN or
   negative norm) the kernel changes nothing: the NaN-safe order K1+K2 -> C1 ->
   K3 leaves every rank's w and m as they were, like the reference, whose
   observe raises (signal.py:67-68) before sgd_step runs (strategies.py:286, :383).
   With mu = wd = 0 this is sgd_step (model.py:215-221); s = 1/N pre-scales the
   parameters for an allreduce-SUM (the 1/N of aggregate_mean, strategies.py:167).
   m_dev may be NULL when momentum == 0. */
SS_API int ss_sgd_update_f32(float* w_dev, const float* g_dev, float* m_dev, int64_t n, float lr,
                      float momentum, float dampening, float weight_decay, int32_t nesterov,
                      int32_t first_step, const int32_t* sync_word_dev, float sync_scale,
                      void* stream);

/* K13+K2: the fused parameter-aggregation step of _selsync_step
   (strategies.py:378-384): one pass reads w, g, m and writes w, m while
   accumulating ||g||^2; the finishing block runs the signal step and writes
   the flag word. 20P bytes with momentum, 12P without. */
SS_API int ss_update_norm_signal_f32(float* w_dev, const float* g_dev, float* m_dev, int64_t n, float lr,
                              float momentum, float dampening, float weight_decay,
                              int32_t nesterov, int32_t first_step, ss_signal_state* st_dev,
                              double delta, int32_t* word_dev, ss_trace_row* trace_dev,
                              int32_t trace_cap, void* ws_dev, void* stream);

/* K3 / K13+K2 over a LIST of tensors (no flat buffer): HOST arrays of device
   pointers w[k], g[k], m[k] (m may be NULL when momentum == 0) and sizes[k].
   Same arithmetic as ss_sgd_update_f32 / ss_update_norm_signal_f32; the norm
   covers all tensors and finishes deterministically in one block (one logical
   launch per <= 128 tensors). */
SS_API int ss_sgd_update_multi_f32(float* const* w_host, const float* const* g_host, float* const* m_host,
                                   const int64_t* sizes_host, int32_t count, float lr, float momentum,
                                   float dampening, float weight_decay, int32_t nesterov, int32_t first_step,
                                   const int32_t* sync_word_dev, float sync_scale, void* stream);
SS_API int ss_update_norm_signal_multi_f32(float* const* w_host, const float* const* g_host,
                                           float* const* m_host, const int64_t* sizes_host, int32_t count,
                                           float lr, float momentum, float dampening, float weight_decay,
                                           int32_t nesterov, int32_t first_step, ss_signal_state* st_dev,
                                           double delta, int32_t* word_dev, ss_trace_row* trace_dev,
                                           int32_t trace_cap, void* ws_dev, void* stream);

/* ---------------- simulated workers on one device ---------------- */

/* aggregate_mean (strategies.py:159-168) over `count` replica buffers in
   index order, result written back into every buffer (the PS broadcast of
   runtime.py:285-287). bufs_host: HOST array of device pointers, count <= 64. */
SS_API int ss_replica_average_f32(float* const* bufs_host, int32_t count, int64_t n, void* stream);

/* the same reduction without the division: the allreduce-SUM that follows
   a 1/N pre-scale in the update epilogue (ss_sgd_update_f32 sync_scale) */
SS_API int ss_replica_sum_f32(float* const* bufs_host, int32_t count, int64_t n, void* stream);

/* elementwise mean of `count` buffers into out_dev (may alias a source) */
SS_API int ss_mean_f32(const float* const* bufs_host, int32_t count, int64_t n, float* out_dev,
                void* stream);

/* flag exchange of runtime.py:319-333 for replicas: max over the words,
   written back to every word. words_host: HOST array of device pointers. */
SS_API int ss_replica_flag_max_i32(int32_t* const* words_host, int32_t count, void* stream);

/* ---------------- device-side exchange over NVLink peer memory ---------------- */

#define SS_SYMM_MAX_RANKS 16
#define SS_SYMM_ERR_TIMEOUT 1

/* A rank's view of the symmetric (peer-mapped) parameter buffer and of every
   rank's signal region. Filled once by the host (e.g. from
   torch.distributed._symmetric_memory.rendezvous); all pointers are device
   addresses valid in this process. The signal regions hold 3*world uint64
   slots (ss_symm_signal_bytes: votes double-buffered by step parity + end-
   barrier tags) and must start zeroed on every rank. */
#define SS_ORDER_MODE_MASK 0x3          /* order_mode bits selecting order 0-3 */
#define SS_ORDER_EARLY_VOTE 0x10        /* order_mode flag: the exact early vote (opt-in) */

typedef struct ss_symm_group {
    float* bufs[SS_SYMM_MAX_RANKS];     /* rank r's flat fp32 buffer */
    uint64_t* pads[SS_SYMM_MAX_RANKS];  /* rank r's signal region */
    float* mc;                          /* multicast (NVLS) address of the buffer, or NULL */
    uint32_t* seq;                      /* step counter, zero-initialised, advanced by the kernels */
    int32_t* agreed_ring;               /* optional ring of agreed words, one per step */
    int32_t* err;                       /* set to SS_SYMM_ERR_TIMEOUT when a peer does not answer */
    double timeout_s;                   /* bound of every spin (> 0) */
    int32_t rank;
    int32_t world;
    int32_t ring_cap;
    int32_t max_blocks;                 /* cap on the grid of the one-launch step kernels (0 = one full
                                           wave: #SMs x resident blocks). Ranks that share ONE device
                                           (colocated ranks) split it: every rank's grid must be
                                           co-resident with every other rank's at once. */
    /* order of the one-launch step (ss_step_symm_f32):
         0  update first: K13 (update + ||g||^2) then, on sync, the mean;
         1  norm first: K1, vote, then on sync ONE kernel that overlaps the update
            of each tile with the NVLink mean of tiles all ranks have finished
            (on local steps the plain update);
         2  adaptive: order 1 when the predicted sync probability >= threshold (EWMA of
            the agreed decisions per context of the previous two);
         3  NaN-safe: order 1 in which the updates wait for the agreed vote, so a
            step on which any rank observed a NaN norm (signal.py:67-68, raised
            before sgd_step at strategies.py:286 vs :383) changes no rank's
            parameters or momentum (SignalError on every rank).
       Orders 1/2 with tile_norm also run the known-sync pass on steps whose
       decision is sync before ||g||^2 is known (ss_sync_known_ahead); a rank
       whose update tile holds a NaN poisons the mean of that tile on its owner,
       so a NaN never reaches another rank's buffer.
       order_mode | SS_ORDER_EARLY_VOTE (orders 1/2 outside the known pass, opt-in):
       the exact early vote -- the ||g||^2 sweep reports a running sum in 8
       chunks, and once that lower bound proves the vote sync
       (ss_sync_proven_early: an upward jump) an early tag lets every rank's
       mean tickets start before the sweep ends; a NaN update tile then
       poisons its mean as in the known pass. Measured: no gain.
       All orders compute identical parameters. Orders 1-3 need the fields below. */
    int32_t order_mode;
    float order_threshold;
    uint32_t* tile_cnt[SS_SYMM_MAX_RANKS]; /* rank r's per-tile arrival counters (peer-mapped, zeroed) */
    uint32_t* epoch;                    /* overlapped sync steps completed (zeroed) */
    float* predictor;                   /* 5 floats, zeroed: P(sync) EWMA per context of the
                                           last two agreed decisions, then the context */
    int64_t tile_elems;                 /* elements per tile, multiple of 4 */
    int64_t n_tiles;                    /* capacity of every tile_cnt array */
    double* tile_norm;                  /* optional, n_tiles doubles: per-tile ||g||^2 partials of the
                                           known-sync pass (warmup steps, delta == 0); NULL disables it */
    uint64_t* debug_events;             /* optional: per-ticket timeline of the overlapped step */
    int64_t debug_cap;                  /* tickets recorded (4 x uint64 each) */
} ss_symm_group;

/* bytes of each rank's signal region (2 x world vote slots + world done slots + world
   poison slots + world early-sync slots, uint64 each) */
SS_API int ss_symm_signal_bytes(int32_t world, int64_t* bytes_host);
/* layout check for FFI mirrors of ss_symm_group: byte offsets of its fields in
   declaration order, then sizeof(ss_symm_group); *count_host = entries written
   (fails with SS_ERR_CONFIG when cap is too small) */
SS_API int ss_symm_group_layout(int64_t* offsets_host, int32_t cap, int32_t* count_host);

/* C2 (and optionally C1) as one launch after the update kernel:
     exchange = 1: P2P flag exchange -- the N-bit OR of runtime.py:319-333 as a
                   MAX over seq-tagged words posted into every peer's signal
                   region; *word_dev: own word in, agreed word out;
     exchange = 0: *word_dev already holds the agreed word (NCCL allreduce-MAX).
   If the agreed word is SS_FLAG_SYNC, every rank's buffer is replaced by the
   mean over ranks (runtime.py:275-294, strategies.py:159-168): each rank
   reduces its 1/N shard (multimem.ld_reduce through the NVSwitch when
   g->mc != NULL, else P2P loads in rank order), applies `scale` (= 1/N) in
   the epilogue and stores the result to every rank; an end barrier precedes
   the kernel's exit. The branch is taken on the device: no host round-trip.
   g_host: HOST pointer to the group; ws_dev: a zeroed ss_workspace. */
SS_API int ss_symm_sync_f32(const ss_symm_group* g_host, int64_t n, int32_t* word_dev,
                            int32_t exchange, float scale, void* ws_dev, void* stream);

/* The whole SelSync step in ONE host launch (strategies.py:378-394), issued
   as a cooperative launch (cudaLaunchAttributeCooperative: the driver places
   every block at once or fails the launch -- blocks wait on each other):
   fused update + ||g||^2 (K13) -> signal step in the last block to finish
   (K2) -> its vote posted to every peer -> that block waits for the N votes
   (C1) and broadcasts the agreed word to the other blocks of the grid -> on
   sync, the mean written into every rank's buffer with the 1/N applied in
   the epilogue (C2) -> end barrier. (Orders 1-3: see order_mode.)
   w_dev must be g_host->bufs[g_host->rank]. *word_dev ends as the agreed
   word; the trace row keeps the own vote. SS_ERR_CONFIG when the grid
   (max_blocks) cannot be co-resident. */
SS_API int ss_step_symm_f32(float* w_dev, const float* g_dev, float* m_dev, int64_t n, float lr,
                            float momentum, float dampening, float weight_decay, int32_t nesterov,
                            int32_t first_step, ss_signal_state* st_dev, double delta,
                            int32_t* word_dev, ss_trace_row* trace_dev, int32_t trace_cap,
                            const ss_symm_group* g_host, void* ws_dev, void* stream);

/* The gradient-aggregation step in one launch (strategies.py:395-399 with
   the server's GA round, runtime.py:259-273): ||g||^2 + vote, then on sync
   the mean GRADIENT over ranks (tile by tile, NVLS / P2P) and the update with
   it; on local steps the update with the own gradient. g_dev must be
   g_host->bufs[g_host->rank] (the gradient lives in symmetric memory);
   needs tile_cnt / epoch / tile_elems of the group. The vote precedes every
   update here, so an agreed word with an error bit (a NaN on any rank)
   leaves every rank's parameters and momentum untouched. Cooperative launch. */
SS_API int ss_step_symm_ga_f32(float* w_dev, float* g_dev, float* m_dev, int64_t n, float lr,
                               float momentum, float dampening, float weight_decay, int32_t nesterov,
                               int32_t first_step, ss_signal_state* st_dev, double delta,
                               int32_t* word_dev, ss_trace_row* trace_dev, int32_t trace_cap,
                               const ss_symm_group* g_host, void* ws_dev, void* stream);

/* ---------------- ranks sharing one device (colocated) ---------------- */

/* One rank's arguments of ss_step_symm_f32 / ss_step_symm_ga_f32 except the
   per-step lr and first-step flag. group is a HOST pointer read by prepare. */
typedef struct ss_rank_step {
    float* w_dev;
    float* g_dev;
    float* m_dev;
    int64_t n;
    float momentum;
    float dampening;
    float weight_decay;
    int32_t nesterov;
    ss_signal_state* st_dev;
    double delta;
    int32_t* word_dev;
    ss_trace_row* trace_dev;
    int32_t trace_cap;
    int32_t reserved;
    const ss_symm_group* group;
    void* ws_dev;
} ss_rank_step;

typedef struct ss_colocated_plan {
    void* args_dev;           /* in: caller-owned device buffer of ss_colocated_args_bytes(ranks) bytes */
    int32_t ranks;            /* out */
    int32_t blocks_per_rank;  /* out: G, each rank's slice of the launch */
    int32_t grads;            /* out: 1 = gradient aggregation (ss_step_symm_ga_f32's kernel) */
    int32_t flags;            /* out: bit 0 momentum, bit 1 Nesterov */
} ss_colocated_plan;

/* N ranks on ONE device (N = 1, 2, 4, 8; every rank's ss_symm_group holds the
   other ranks' same-device buffers as its peers, mc = NULL) step together in
   ONE cooperative launch of N x G blocks: blocks [r*G, (r+1)*G) run rank r's
   one-launch step (the kernels of ss_step_symm_f32 / _ga_f32, bit-identical
   work per rank) -- never as N launches that wait on one another, which
   nothing guarantees to run at the same time. This is the reference's
   N-worker round (runtime.py:275-294, :319-333) on a single GPU.
   prepare validates every rank (as ss_step_symm_f32 does), picks G (the
   rank's one-wave grid, capped so all N grids are co-resident; optionally
   by max_blocks_per_rank) and copies the argument blocks into
   plan->args_dev (synchronous on `stream`); step launches one step of all
   ranks (CUDA-graph capturable). */
SS_API int ss_colocated_args_bytes(int32_t ranks, int64_t* bytes_host);
SS_API int ss_colocated_prepare_f32(const ss_rank_step* ranks_host, int32_t ranks, int32_t grads,
                                    int32_t max_blocks_per_rank, ss_colocated_plan* plan_host, void* stream);
SS_API int ss_colocated_step_f32(const ss_colocated_plan* plan_host, float lr, int32_t first_step, void* stream);

/* ---------------- prepared per-rank step (the lean per-step host path) ---------------- */

/* One rank's step with everything but the gradient pointer, lr and the
   first-step flag validated once. init checks what the per-call entry points
   check on every call -- group == NULL: one rank, ss_update_norm_signal_f32
   (K13+K2); otherwise ss_step_symm_f32, or ss_step_symm_ga_f32 when grads = 1
   -- picks the kernel and keeps its argument blocks in the caller's plan;
   launch patches g_dev, lr and first_step and issues the same launch
   (cooperative for the group kernels; CUDA-graph capturable). The group is
   read at init: re-init after changing it. This is the per-step call of
   _selsync_step (strategies.py:369-403) made as one 5-argument C call: a
   step of a small model is shorter than marshalling the 18 arguments of the
   per-call entry points (1M parameters: ~8 us of GPU work per step). */
#define SS_STEP_PLAN_WORDS 192
typedef struct ss_step_plan {
    uint64_t opaque[SS_STEP_PLAN_WORDS];
} ss_step_plan;
SS_API int ss_step_plan_init(ss_step_plan* plan_host, const ss_rank_step* rank_host, int32_t grads);
SS_API int ss_step_plan_launch(const ss_step_plan* plan_host, const float* g_dev, float lr, int32_t first_step,
                               void* stream);
/* Compiled field offsets of ss_rank_step in declaration order, then
   sizeof(ss_rank_step) and sizeof(ss_step_plan): lets a binding check its
   mirror of the structs (host-only, no GPU). */
SS_API int ss_rank_step_layout(int64_t* offsets_host, int32_t cap, int32_t* count_host);

#ifdef __cplusplus
}
#endif

#endif /* SELSYNC_B200_H */
