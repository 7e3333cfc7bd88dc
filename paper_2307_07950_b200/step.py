"""``SelSyncStep`` -- one rank's selective-synchronization step on a B200.

Mirrors ``_selsync_step`` (strategies.py:369-403) for the caller that used to
be ``run_worker`` + the parameter server: a per-rank training loop that calls
``step(lr)`` after ``loss.backward()`` has written the flat gradient buffer.

Order of device work per step (parameter aggregation, the default):

  K13+K2  one kernel: local update w, m <- SGD(w, g, m) (the reference applies
          it before the vote, :380-383) while reducing ||g||^2 in fp64; the
          finishing block runs observe/relative_change/decide on the device
          state and writes the int32 flag word          (:378-384, signal.py)
  C1      NCCL allreduce-MAX of the flag word = OR of the N votes
                                                        (runtime.py:319-333)
  C2      on sync only: NCCL allreduce-AVG of the flat fp32 parameters
                                                        (runtime.py:275-294)

``fuse=False`` selects the pre-scale order instead: K1+K2, C1, then K3 whose
epilogue multiplies the updated parameters by 1/N when the agreed word says
sync, then allreduce-SUM. Its host read of the word overlaps K3.

Gradient aggregation (``aggregation="grads"``, :395-399): K1+K2, C1, then on
sync allreduce-AVG of the gradients before the update, else the own gradient.

The host learns the agreed decision through a 4-byte pinned copy of the word
(an event wait); that is the only host<->device traffic of a step.
"""

from __future__ import annotations

from typing import Optional

import math

import torch

from . import kernels as K
from .collectives import RankGroup
from .config import SelSyncConfig
from .errors import ConfigError, SignalError


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
        trace_capacity: int = 4096,
        broadcast_init: bool = True,
        profile: bool = False,
    ):
        if not isinstance(config, SelSyncConfig):
            raise ConfigError("config must be a SelSyncConfig")
        K._need(params, torch.float32, "params")
        K._need(grads, torch.float32, "grads", params.device)
        if params.dim() != 1 or grads.shape != params.shape:
            raise ConfigError("params and grads must be flat fp32 vectors of the same length")
        self.config = config
        self.device = params.device
        self.params = params
        self.grads = grads
        self.comm = group if isinstance(group, RankGroup) else RankGroup(group)
        self.world = self.comm.size
        self.worker_id = self.comm.rank
        self.fuse = bool(fuse) and config.aggregation == "params"
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
        self._word_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._ready = torch.cuda.Event()
        self.steps_done = 0
        self.decisions: list[bool] = []
        self.lrs: list[float] = []
        self.profile = profile
        self.kernel_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        self.sync_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        if broadcast_init and self.world > 1:
            self.comm.broadcast_(self.params, 0)

    # ------------------------------------------------------------------
    def _events(self, bucket):
        if not self.profile:
            return None
        pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        bucket.append(pair)
        return pair

    def _read_word(self, stream) -> int:
        self._word_host.copy_(self.signal.word, non_blocking=True)
        self._ready.record(stream)
        return 0

    def step(self, lr: float) -> str:
        """Run one SelSync step on the gradients currently in ``grads``.

        Returns the agreed decision, ``"sync"`` or ``"local"``. Raises
        SignalError on every rank if any rank observed a NaN norm."""
        lr = float(lr)
        if not (lr >= 0.0) or not math.isfinite(lr):
            raise ConfigError(f"learning rate must be non-negative, got {lr}")
        cfg = self.config
        first = self.steps_done == 0
        stream = torch.cuda.current_stream(self.device)
        hp = dict(momentum=cfg.momentum, dampening=cfg.dampening, weight_decay=cfg.weight_decay,
                  nesterov=cfg.nesterov, first_step=first)
        ev = self._events(self.kernel_events)
        if ev:
            ev[0].record(stream)
        if self.fuse:
            K.update_norm_signal_(self.params, self.grads, self.momentum, self.signal, self.ws,
                                  lr=lr, delta=cfg.delta, **hp)
        else:
            K.norm_signal(self.grads, self.signal, cfg.delta, self.ws)
        if ev:
            ev[1].record(stream)
        self.comm.agree(self.signal.word)
        self._read_word(stream)
        if cfg.aggregation == "params" and not self.fuse:
            # the host read above overlaps this update
            K.sgd_update_(self.params, self.grads, self.momentum, lr=lr,
                          sync_word=self.signal.word, sync_scale=1.0 / self.world, **hp)
        self._ready.synchronize()
        word = int(self._word_host[0])
        if word >= 2:
            K.raise_for_word(word, f" (agreed flag word {word} at step {self.steps_done})")
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
            K.sgd_update_(self.params, self.grads, self.momentum, lr=lr, **hp)
        self.steps_done += 1
        self.decisions.append(synced)
        self.lrs.append(lr)
        return "sync" if synced else "local"

    # ------------------------------------------------------------------
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
        out = []
        for step in range(max(0, self.steps_done - cap), self.steps_done):
            r = rows[step % cap]
            d = float(r["delta_g"])
            out.append(dict(
                step=step, worker_id=self.worker_id, grad_norm_sq=float(r["grad_norm_sq"]),
                ewma=float(r["ewma"]), delta_g=None if math.isnan(d) else d,
                decision="sync" if self.decisions[step] else "local",
                vote=bool(int(r["word"]) & 1), lr=self.lrs[step]))
        return out

    def kernel_ms(self) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.kernel_events]

    def sync_ms(self) -> list[float]:
        return [a.elapsed_time(b) for a, b in self.sync_events]
