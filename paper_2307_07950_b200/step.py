"""``SelSyncStep`` -- one rank's selective-synchronization step on a B200.

Mirrors ``_selsync_step`` (strategies.py:369-403) for the caller that used to
be ``run_worker`` + the parameter server: a per-rank training loop calling
``step(lr)`` after ``loss.backward()`` has filled the flat gradient buffer.

Device work per step, parameter aggregation (the default):

  K13+K2  one kernel: the local update w, m <- SGD(w, g, m) (the reference
          applies it before the vote, :380-383) while reducing ||g||^2 in
          fp64; the finishing block runs observe / relative_change / decide
          on the device-resident state and writes the int32 flag word
  C1      allreduce-MAX of the flag word = OR of the N votes (runtime.py:319-333)
          -- a seq-tagged P2P exchange over NVLink inside the step kernel
          (default), or an NCCL allreduce-MAX of the word
  C2      sync steps only: the parameter mean (runtime.py:275-294)

Back ends (N > 1):
  collective="symm" (default): parameters live in symmetric memory.
      flag_exchange="fused" (default): the whole step is ONE cooperative launch
      (``ss_step_symm_f32``): update + norm + vote, the vote exchange over
      NVLink in the last block to finish, which broadcasts the agreed word to
      the rest of the grid; on sync every block then runs its part of the
      mean (NVLS multimem or P2P, 1/N in the epilogue) and the last one the
      end barrier -- no second launch. ``order`` picks update-first,
      norm-first (update and mean overlapped tile by tile), adaptive, or
      nan_safe (norm-first with the updates waiting for the vote).
      flag_exchange="p2p" / "nccl": K13, then ``ss_symm_sync_f32`` reading the
      agreed word (its own P2P exchange, or an NCCL allreduce-MAX before it).
      No host round-trip in any of them: ``step_async`` enqueues a whole step
      and returns; the host reads decisions lazily.
  collective="nccl": the host reads the agreed word (4-byte pinned copy) and
      issues NCCL allreduce-AVG on sync steps. ``fuse=False`` selects the
      pre-scale order instead: K1+K2, C1, K3 whose epilogue multiplies by 1/N
      when the agreed word says sync (the host read overlaps K3), allreduce-SUM.
  Ranks sharing one GPU (``colocated.ColocatedSelSync``) run the same step
  kernels over same-device buffers, all ranks in ONE cooperative launch (rank
  r's blocks are slice r of the grid).

Gradient aggregation (aggregation="grads", :395-399): over symmetric memory
the one-launch ``ss_step_symm_ga_f32`` (norm + vote, then per tile the
owner's mean of the GRADIENT and the update with it); on the NCCL back end
K1+K2, C1, then on sync allreduce-AVG of the gradients, then the update.

NaN semantics (``nan_safe=True``): the reference raises in observe
(signal.py:67-68) before sgd_step (strategies.py:286 vs :383), so a NaN step
mutates nothing. The fused update + norm pass updates before it knows the
norm; with nan_safe the step uses an order in which every update waits for
the agreed word and skips on an error bit (K1+K2 -> C1 -> K3, or the
one-launch "nan_safe" order). Without it, only the rank that met the NaN is
affected: no mean ever carries a NaN to another rank (the vote, or in the
known-sync pass a per-tile poison tag, stops it), and SignalError is raised
on every rank.
"""

from __future__ import annotations

import ctypes
import math
from collections import deque
from typing import Optional

import torch

from . import _native as N
from . import kernels as K
from .collectives import RankGroup, resolve_order
from .config import SelSyncConfig
from .errors import ConfigError

_PLAN_LAUNCH = N.LIB.ss_step_plan_launch


class SelSyncStep:
    def __init__(
        self,
        params: torch.Tensor,
        grads: torch.Tensor,
        config: SelSyncConfig,
        *,
        momentum_buffer: Optional[torch.Tensor] = None,
        group=None,
        fuse: bool = True,
        collective: Optional[str] = None,
        flag_exchange: Optional[str] = None,
        trace_capacity: int = 4096,
        broadcast_init: bool = True,
        profile: bool = False,
        timeout_s: float = 10.0,
        order: str = "auto",
        order_threshold: float = 0.2,
        tile_elems: Optional[int] = None,
        multicast="auto",
        nan_safe: bool = False,
        max_blocks: int = 0,
        early_vote: bool = False,
    ):
        if not isinstance(config, SelSyncConfig):
            raise ConfigError("config must be a SelSyncConfig")
        K._need(params, torch.float32, "params")
        K._need(grads, torch.float32, "grads", params.device)
        if params.dim() != 1 or grads.shape != params.shape:
            raise ConfigError("params and grads must be flat fp32 vectors of the same length")
        self.config = config
        self.device = params.device
        self.grads = grads
        # a RankGroup, a rank group of ranks sharing one device (colocated), or a
        # torch.distributed process group (None = WORLD)
        self.comm = group if isinstance(group, RankGroup) or hasattr(group, "make_symmetric") else RankGroup(group)
        self.world = self.comm.size
        self.worker_id = self.comm.rank
        colocated = self.comm.backend == "colocated"
        if collective is None:
            collective = "symm" if colocated or (self.world > 1 and config.aggregation == "params"
                                                 and self.comm.backend == "nccl") else "nccl"
        if colocated and collective != "symm":
            raise ConfigError("colocated ranks exchange through the symmetric-memory step (collective='symm')")
        if collective not in ("nccl", "symm"):
            raise ConfigError(f"collective must be 'nccl' or 'symm', got {collective!r}")
        if flag_exchange is None:
            flag_exchange = "fused" if collective == "symm" else "nccl"
        if flag_exchange not in ("nccl", "p2p", "fused"):
            raise ConfigError(f"flag_exchange must be 'fused', 'p2p' or 'nccl', got {flag_exchange!r}")
        if flag_exchange in ("p2p", "fused") and collective != "symm" and self.world > 1:
            raise ConfigError("the P2P flag exchange runs inside the symmetric-memory kernels")
        # one rank: no exchange -- unless symmetric memory is asked for explicitly
        # (the one-launch kernel on a single GPU, e.g. to profile it under ncu)
        self.collective = collective if (self.world > 1 or collective == "symm"
                                        and (colocated or torch.distributed.is_initialized())) else "none"
        self.flag_exchange = flag_exchange
        # "auto": adaptive where the overlapped norm-first pass pays, else update-first
        order = resolve_order(order, params.numel(), self.world)
        # NaN-safe: a step on which any rank observes a NaN norm changes no
        # rank's parameters (the reference raises in observe, signal.py:67-68,
        # before sgd_step, strategies.py:286 vs :383). The fused update + norm
        # pass cannot promise that, so it gives way to K1+K2 -> C1 -> K3 (the
        # pre-scale order, K3 skipping on an error word) or, over symmetric
        # memory, to the one-launch step's "nan_safe" order.
        self.nan_safe = bool(nan_safe) or order == "nan_safe"
        if self.nan_safe:
            if self.collective == "symm":
                if flag_exchange != "fused" and config.aggregation == "params":
                    raise ConfigError("nan_safe over symmetric memory is the one-launch step (flag_exchange='fused')")
                order = "nan_safe"
            else:
                fuse = False
        self.fuse = (bool(fuse) or self.collective == "symm") and config.aggregation == "params"
        if self.collective == "symm" and config.aggregation == "grads" and flag_exchange != "fused":
            raise ConfigError("gradient aggregation over symmetric memory is the one-launch step "
                              "(flag_exchange='fused')")
        if config.momentum != 0.0:
            if momentum_buffer is None:
                momentum_buffer = torch.zeros_like(params)
            K._need(momentum_buffer, torch.float32, "momentum_buffer", self.device)
            if momentum_buffer.shape != params.shape:
                raise ConfigError("momentum buffer size does not match parameter vector")
        self.momentum = momentum_buffer if config.momentum != 0.0 else None
        self.smoothing = config.smoothing_for(self.world)
        self.signal = K.DeviceSignal(self.device, self.smoothing, config.warmup, trace_capacity)
        self.ws = K.Workspace(self.device)
        self._fast_cache, self._plans = {}, {}
        self.symm = None
        if self.collective == "symm":
            self.symm = self.comm.make_symmetric(params.numel(), self.device,
                                                 ring_capacity=trace_capacity, timeout_s=timeout_s,
                                                 order=order, order_threshold=order_threshold,
                                                 tile_elems=tile_elems, use_multicast=multicast,
                                                 max_blocks=max_blocks)
            self.symm.set_early_vote(early_vote)
            if config.aggregation == "grads":
                # the exchanged vector is the gradient: it lives in symmetric memory
                self.symm.buf.copy_(grads)
                self.grads = self.symm.buf  # backward must write step.grads
                if not self.symm.one_launch_capable:
                    raise ConfigError(f"gradient aggregation over symmetric memory needs multicast or "
                                      f"2, 4 or 8 ranks (world {self.world})")
            else:
                self.symm.buf.copy_(params)
                params = self.symm.buf  # the step owns the symmetric copy; use step.params
                if self.flag_exchange == "fused" and not self.symm.one_launch_capable:
                    self.flag_exchange = "p2p"
        self.params = params
        self._word_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._ready = torch.cuda.Event()
        self.steps_done = 0
        # host-side per-step log, bounded to the trace-ring window (records() /
        # decisions() cover the last trace_capacity steps): decisions the host
        # learned in blocking steps, and the lr of every step
        self._host_decisions: dict[int, bool] = {}
        self._lr_ring: list[float] = [0.0] * self.signal.trace_capacity
        self.profile = profile
        self.kernel_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        self.sync_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        if broadcast_init and self.world > 1:
            self.comm.broadcast_(self.params, 0)

    # ------------------------------------------------------------------
    @property
    def async_capable(self) -> bool:
        """True when a step never needs the host to learn the branch."""
        return self.collective == "symm" or (self.collective == "none" and self.fuse)

    def _events(self, bucket):
        if not self.profile:
            return None
        pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        bucket.append(pair)
        return pair

    def _hp(self, first: bool) -> dict:
        c = self.config
        return dict(momentum=c.momentum, dampening=c.dampening, weight_decay=c.weight_decay,
                    nesterov=c.nesterov, first_step=first)

    def _check_lr(self, lr) -> float:
        lr = float(lr)
        if not (lr >= 0.0) or not math.isfinite(lr):
            raise ConfigError(f"learning rate must be non-negative, got {lr}")
        return lr

    def _wait_word(self, stream) -> int:
        self._word_host.copy_(self.signal.word, non_blocking=True)
        self._ready.record(stream)
        self._ready.synchronize()
        word = int(self._word_host[0])
        if word >= 2:
            K.raise_for_word(word, f" (agreed flag word {word} at step {self.steps_done})")
        return word

    def _enqueue_device_step(self, lr: float, stream) -> None:
        """K13+K2 -> C1 -> conditional C2, entirely on the device."""
        if self.comm.backend == "colocated" and self.world > 1:
            raise ConfigError("colocated ranks step together in one launch: use ColocatedSelSync.step")
        cfg = self.config
        ev = self._events(self.kernel_events)
        if ev:
            ev[0].record(stream)
        if self.collective == "symm" and self.flag_exchange == "fused":
            # one host launch: update, norm, vote, vote exchange, conditional mean
            self._fast_launch("symm_ga" if cfg.aggregation == "grads" else "symm", lr, stream)
            if ev:
                ev[1].record(stream)
            return
        self._fast_launch("k13", lr, stream)
        if ev:
            ev[1].record(stream)
        if self.collective == "symm":
            ev = self._events(self.sync_events)
            if ev:
                ev[0].record(stream)
            if self.flag_exchange == "nccl":
                self.comm.agree(self.signal.word)
            self.symm.sync_(self.signal.word, self.ws.ptr, exchange=self.flag_exchange == "p2p",
                            stream=stream.cuda_stream)
            K._count()
            if ev:
                ev[1].record(stream)

    def _fast_launch(self, which: str, lr: float, stream) -> None:
        """Launch K13+K2 (or the one-launch symmetric step) through a prepared
        step plan (``ss_step_plan_init``: every argument validated once); per
        step only the gradient pointer (the caller may rebind ``grads``), lr
        and the first-step flag cross into C, in one 5-argument call. At small
        P a step is shorter than the host path, so this path is kept short."""
        g = self.grads
        key = (which, id(g), g.data_ptr(), g.numel(), self.symm.version if self.symm is not None else 0)
        entry = self._fast_cache.get(key)
        if entry is None:
            entry = self._prepare_launch(which, g, key)
        rc = _PLAN_LAUNCH(entry[0], entry[1], lr, self.steps_done == 0, stream.cuda_stream)
        if rc:
            N.check(rc)
        K._count()

    def _prepare_launch(self, which: str, g: torch.Tensor, key):
        # full validation whenever a gradient buffer is bound for the first
        # time (a training loop may rotate a few buffers; each is checked once);
        # the entry keeps g alive so its id cannot be reused while cached
        K._sgd_check(self.params, g, self.momentum, self.config.momentum)
        pkey = (which, key[-1])
        plan = self._plans.get(pkey)
        if plan is None:
            c = self.config
            desc = N.RankStepC(
                self.params.data_ptr(), g.data_ptr(),
                self.momentum.data_ptr() if self.momentum is not None else None, self.params.numel(),
                float(c.momentum), float(c.dampening), float(c.weight_decay), int(bool(c.nesterov)),
                self.signal.state.data_ptr(), float(c.delta), self.signal.word.data_ptr(),
                self.signal.trace.data_ptr(), self.signal.trace_capacity, 0,
                ctypes.addressof(self.symm.group_c) if which != "k13" else None, self.ws.ptr)
            plan = N.StepPlanC()
            N.check(N.LIB.ss_step_plan_init(ctypes.addressof(plan), ctypes.addressof(desc),
                                            int(which == "symm_ga")))
            self._plans = {pkey: plan}  # a group change (new version) drops the old plans
        if len(self._fast_cache) >= 16:
            self._fast_cache.clear()
        entry = self._fast_cache[key] = (ctypes.addressof(plan), g.data_ptr(), g, plan)
        return entry

    def step_async(self, lr: float) -> None:
        """Enqueue one whole step and return without waiting for the GPU.
        Needs a device-side branch (world size 1 or collective='symm')."""
        if not self.async_capable:
            raise ConfigError("step_async needs collective='symm' (or a single rank)")
        lr = self._check_lr(lr)
        self._enqueue_device_step(lr, torch.cuda.current_stream(self.device))
        self._log_step(lr)

    def _log_step(self, lr: float, synced: Optional[bool] = None) -> None:
        """Advance the step counter, keeping the host log within the ring window."""
        s, cap = self.steps_done, self.signal.trace_capacity
        if synced is not None:
            self._host_decisions[s] = synced
        self._host_decisions.pop(s - cap, None)
        self._lr_ring[s % cap] = lr
        self.steps_done = s + 1

    def step(self, lr: float) -> str:
        """Run one SelSync step on the gradients in ``grads``; returns the
        agreed decision ``"sync"`` / ``"local"``. Raises SignalError on every
        rank if any rank observed a NaN norm."""
        lr = self._check_lr(lr)
        cfg = self.config
        stream = torch.cuda.current_stream(self.device)
        if self.async_capable:
            self._enqueue_device_step(lr, stream)
            word = self._wait_word(stream)
            if self.symm is not None:
                self.symm.check()
        else:
            first = self.steps_done == 0
            ev = self._events(self.kernel_events)
            if ev:
                ev[0].record(stream)
            if self.fuse:
                K.update_norm_signal_(self.params, self.grads, self.momentum, self.signal, self.ws,
                                      lr=lr, delta=cfg.delta, **self._hp(first))
            else:
                K.norm_signal(self.grads, self.signal, cfg.delta, self.ws)
            if ev:
                ev[1].record(stream)
            self.comm.agree(self.signal.word)
            if cfg.aggregation == "params" and not self.fuse:
                # the host read of the agreed word overlaps this update
                self._word_host.copy_(self.signal.word, non_blocking=True)
                self._ready.record(stream)
                K.sgd_update_(self.params, self.grads, self.momentum, lr=lr,
                              sync_word=self.signal.word, sync_scale=1.0 / self.world, **self._hp(first))
                self._ready.synchronize()
                word = int(self._word_host[0])
                if word >= 2:
                    K.raise_for_word(word, f" (agreed flag word {word} at step {self.steps_done})")
            else:
                word = self._wait_word(stream)
            synced = bool(word & 1)
            if cfg.aggregation == "params":
                if synced and self.world > 1:
                    ev = self._events(self.sync_events)
                    if ev:
                        ev[0].record(stream)
                    if self.fuse:
                        self.comm.average_(self.params)
                    else:
                        self.comm.sum_(self.params)
                    if ev:
                        ev[1].record(stream)
            else:
                if synced and self.world > 1:
                    self.comm.average_(self.grads)
                K.sgd_update_(self.params, self.grads, self.momentum, lr=lr, **self._hp(first))
        synced = bool(word & 1)
        self._log_step(lr, synced)
        return "sync" if synced else "local"

    def capture(self, lr: float, grads_seq=None) -> "CapturedStep":
        """Record one device-branching step (the gradient buffer bound now, this
        lr) as a CUDA graph; ``replay()`` then equals ``step_async(lr)`` at the
        cost of one graph launch. For launch-bound sizes (small P) and loops
        that rotate a fixed set of gradient buffers (capture one per buffer).

        ``grads_seq``: a list of gradient buffers -- one graph then holds
        ``len(grads_seq)`` consecutive steps, step i on ``grads_seq[i]``, and a
        replay advances the step count by that many. Inside one graph each step
        kernel is placed on the SMs while the previous one drains (the
        launches carry programmatic stream serialization), so short steps
        overlap their launch latency."""
        if not self.async_capable:
            raise ConfigError("capture needs a device-side branch (collective='symm' or a single rank)")
        if self.profile:
            raise ConfigError("per-launch profiling events cannot be captured")
        if self.steps_done == 0:
            raise ConfigError("run one eager step first (the first step initialises the momentum buffer)")
        lr = self._check_lr(lr)
        seq = [self.grads] if grads_seq is None else list(grads_seq)
        if not seq:
            raise ConfigError("grads_seq must hold at least one gradient buffer")
        bound = self.grads
        stream = torch.cuda.current_stream(self.device)
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(graph):
                for g in seq:
                    self.grads = g
                    self._enqueue_device_step(lr, torch.cuda.current_stream(self.device))
        finally:
            self.grads = bound
        stream.synchronize()
        return CapturedStep(self, graph, lr, len(seq))

    # ------------------------------------------------------------------
    def synchronize(self) -> None:
        """Wait for enqueued steps; raise on device-side errors (NaN norm, peer timeout)."""
        torch.cuda.current_stream(self.device).synchronize()
        if self.symm is not None:
            self.symm.check()
        s = self.signal.read_state()
        if int(s["error"]):
            K.raise_for_word(int(s["error"]) & 6 or 2, " (device signal state)")
        if self.symm is not None and self.steps_done:
            # a peer's NaN reaches every rank through the agreed word (MAX >= 2)
            cap = self.symm.ring_capacity
            ring = self.symm.agreed.cpu().numpy()
            lo = max(0, self.steps_done - cap)
            bad = [s for s in range(lo, self.steps_done) if int(ring[s % cap]) >= 2]
            if bad:
                K.raise_for_word(int(ring[bad[0] % cap]), f" (agreed flag word at step {bad[0]})")

    def decisions(self) -> list[bool]:
        """Agreed decision of every step still in the trace ring (True = sync)."""
        cap = self.signal.trace_capacity
        lo = max(0, self.steps_done - cap)
        agreed = None
        if self.symm is not None:
            agreed = self.symm.agreed.cpu().numpy()
        own = None
        out = []
        for s in range(lo, self.steps_done):
            if s in self._host_decisions:
                out.append(self._host_decisions[s])
            elif agreed is not None:
                out.append(bool(int(agreed[s % self.symm.ring_capacity]) == 1))
            else:  # single rank: the agreed decision is the own vote
                if own is None:
                    own = self.signal.read_trace()
                out.append(bool(int(own[s % cap]["word"]) & 1))
        return out

    def signal_state(self):
        """Host copy of the device GradSignalState (signal.py:41-61)."""
        from .signal import GradSignalState

        s = self.signal.read_state()
        return GradSignalState(
            smoothing=float(s["smoothing"]), warmup=int(s["warmup"]),
            ewma_current=float(s["ewma_current"]), ewma_previous=float(s["ewma_previous"]),
            step_count=int(s["step_count"]), max_delta_seen=float(s["max_delta_seen"]))

    def records(self) -> list[dict]:
        """Per-step rows in the MetricsRecord schema (metrics.py:23-48) for the
        steps still held by the device trace ring."""
        rows = self.signal.read_trace()
        cap = self.signal.trace_capacity
        dec = self.decisions()
        lo = max(0, self.steps_done - cap)
        out = []
        for i, step in enumerate(range(lo, self.steps_done)):
            r = rows[step % cap]
            d = float(r["delta_g"])
            out.append(dict(
                step=step, worker_id=self.worker_id, grad_norm_sq=float(r["grad_norm_sq"]),
                ewma=float(r["ewma"]), delta_g=None if math.isnan(d) else d,
                decision="sync" if dec[i] else "local",
                vote=bool(int(r["word"]) & 1), lr=self._lr_ring[step % cap]))
        return out

    def kernel_ms(self) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.kernel_events]

    def sync_ms(self) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.sync_events]


class CapturedStep:
    """A SelSync step recorded as a CUDA graph (``SelSyncStep.capture``)."""

    def __init__(self, step: SelSyncStep, graph, lr: float, steps: int = 1):
        self.step, self.graph, self.lr, self.steps = step, graph, lr, steps

    def replay(self) -> None:
        self.graph.replay()
        for _ in range(self.steps):
            self.step._log_step(self.lr)
            K._count()


class TensorListSelSyncStep:
    """SelSync step over a LIST of parameter / gradient tensors (no flat
    buffer): K13+K2 over a pointer table (``ss_update_norm_signal_multi_f32``,
    ||g||^2 of the whole model in one logical launch), C1 as an NCCL
    allreduce-MAX of the flag word, and on sync steps the parameter mean as
    NCCL allreduce-AVG over the tensors, coalesced into one NCCL group.

    Use it when the model's storage cannot be re-pointed at flat buffers;
    ``SelSyncStep`` over ``FlatParameters`` is the faster path.
    """

    def __init__(self, params, grads, config: SelSyncConfig, *, momentum_buffers=None, group=None,
                 trace_capacity: int = 4096, broadcast_init: bool = True):
        if not isinstance(config, SelSyncConfig):
            raise ConfigError("config must be a SelSyncConfig")
        if config.aggregation != "params":
            raise ConfigError("TensorListSelSyncStep implements parameter aggregation")
        self.params, self.grads = list(params), list(grads)
        if not self.params or len(self.params) != len(self.grads):
            raise ConfigError("params and grads must be non-empty lists of equal length")
        self.config = config
        self.device = self.params[0].device
        if config.momentum != 0.0 and momentum_buffers is None:
            momentum_buffers = [torch.zeros_like(p) for p in self.params]
        self.momentum = list(momentum_buffers) if config.momentum != 0.0 else None
        self.comm = group if isinstance(group, RankGroup) else RankGroup(group)
        self.world = self.comm.size
        self.signal = K.DeviceSignal(self.device, config.smoothing_for(self.world), config.warmup,
                                     trace_capacity)
        self.ws = K.Workspace(self.device)
        self._word_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._ready = torch.cuda.Event()
        self.steps_done = 0
        self.decision_log: deque = deque(maxlen=trace_capacity)  # last trace_capacity decisions
        if broadcast_init and self.world > 1:
            for p in self.params:
                self.comm.broadcast_(p, 0)

    def _average(self) -> None:
        import torch.distributed as dist

        try:
            from torch.distributed.distributed_c10d import _coalescing_manager
        except ImportError:  # pragma: no cover - older torch
            _coalescing_manager = None
        if _coalescing_manager is not None and self.comm.backend == "nccl":
            with _coalescing_manager(group=self.comm.group, device=self.device):
                for p in self.params:
                    dist.all_reduce(p, op=dist.ReduceOp.AVG, group=self.comm.group)
        else:
            for p in self.params:
                self.comm.average_(p)

    def step(self, lr: float) -> str:
        lr = float(lr)
        if not (lr >= 0.0) or not math.isfinite(lr):
            raise ConfigError(f"learning rate must be non-negative, got {lr}")
        c = self.config
        K.update_norm_signal_multi_(self.params, self.grads, self.momentum, self.signal, self.ws, lr=lr,
                                    delta=c.delta, momentum=c.momentum, dampening=c.dampening,
                                    weight_decay=c.weight_decay, nesterov=c.nesterov,
                                    first_step=self.steps_done == 0)
        self.comm.agree(self.signal.word)
        self._word_host.copy_(self.signal.word, non_blocking=True)
        self._ready.record(torch.cuda.current_stream(self.device))
        self._ready.synchronize()
        word = int(self._word_host[0])
        if word >= 2:
            K.raise_for_word(word, f" (agreed flag word {word} at step {self.steps_done})")
        synced = bool(word & 1)
        if synced and self.world > 1:
            self._average()
        self.steps_done += 1
        self.decision_log.append(synced)
        return "sync" if synced else "local"
