"""Per-rank SelSync training loop over a model workload.

The caller side of the hot path: zero the flat gradient buffer, stock PyTorch
forward/backward (gradients land in the flat buffer through the ``p.grad``
views), then one ``SelSyncStep``. This replaces the reference's
``run_worker`` + parameter-server loop (strategies.py:487-517,
runtime.py:462-581) for real models on B200s.
"""

from __future__ import annotations

from typing import Optional

import torch

from .config import SelSyncConfig
from .model import FlatParameters
from .step import SelSyncStep
from .workloads import Workload


class SelSyncTrainer:
    """Per-rank loop: forward/backward into the flat gradient, then the
    SelSync step. Besides the device decision trace it keeps, per iteration,
    the loss (a device ring, no host sync) and the iteration's device time
    (CUDA events around forward + backward + step), so ``metrics_rows()``
    fills the reference's ``loss`` and ``step_duration`` columns
    (strategies.py:326-339, metrics.py:23-48; the reference's duration is the
    wall time of the step, strategies.py:298-302)."""

    def __init__(self, workload: Workload, *, delta: float, warmup: int = 25,
                 smoothing: Optional[float] = None, group=None, record_metrics: bool = True, **step_kw):
        self.wl = workload
        self.flat = FlatParameters(workload.model.parameters())
        cfg = SelSyncConfig(delta=delta, warmup=warmup, smoothing=smoothing,
                            momentum=workload.momentum, weight_decay=workload.weight_decay)
        self.step = SelSyncStep(self.flat.params, self.flat.grads, cfg, group=group, **step_kw)
        if self.step.params.data_ptr() != self.flat.params.data_ptr():
            self.flat.rebind(self.step.params)  # parameters now live in symmetric memory
        if self.step.grads.data_ptr() != self.flat.grads.data_ptr():
            self.flat.rebind_grads(self.step.grads)  # gradient aggregation: grads in symmetric memory
        self.iteration = 0
        self.record_metrics = bool(record_metrics)
        cap = self.step.signal.trace_capacity
        self._loss_ring = torch.full((cap,), float("nan"), dtype=torch.float32, device=self.step.device)
        self._events: dict[int, tuple] = {}  # iteration -> (start, end) events, last `cap` iterations

    def _begin(self):
        if not self.record_metrics:
            return None
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record(torch.cuda.current_stream(self.step.device))
        return ev

    def _end(self, ev, loss: torch.Tensor) -> None:
        if ev is None:
            return
        cap = self._loss_ring.numel()
        self._loss_ring[self.iteration % cap].copy_(loss.reshape(()), non_blocking=True)
        ev[1].record(torch.cuda.current_stream(self.step.device))
        self._events[self.iteration] = ev
        self._events.pop(self.iteration - cap, None)

    def forward_backward(self, batch=None) -> torch.Tensor:
        if batch is None:
            batch = self.wl.make_batch(self.iteration)
        self.flat.zero_grad()
        loss = self.wl.loss(self.wl.model, batch)
        loss.backward()
        return loss.detach()

    def train_step(self, batch=None, *, wait: bool = False):
        """One iteration; returns (loss tensor, decision or None when wait=False
        and the step branches on the device)."""
        ev = self._begin()
        loss = self.forward_backward(batch)
        lr = self.wl.lr(self.iteration)
        if wait or not self.step.async_capable:
            decision = self.step.step(lr)
        else:
            self.step.step_async(lr)
            decision = None
        self._end(ev, loss)
        self.iteration += 1
        return loss, decision

    # ------------------------------------------------------------------ graphs
    def capture(self, batch, warmup_iters: int = 3) -> None:
        """Capture forward + backward + the SelSync device step into ONE CUDA
        graph over static batch tensors (``batch`` is (inputs, targets) on the
        device; refill them in place before every ``replay_step``). Needs a
        device-side branch (one rank, or collective="symm"). The learning rate
        is a kernel argument: a new lr re-captures."""
        from .errors import ConfigError

        if not self.step.async_capable:
            raise ConfigError("graph capture needs the device-side branch (one rank or collective='symm')")
        if self.step.profile:
            raise ConfigError("per-launch profiling events cannot be captured")
        self.static_batch = tuple(batch)
        side = torch.cuda.Stream(self.step.device)
        side.wait_stream(torch.cuda.current_stream(self.step.device))
        with torch.cuda.stream(side):  # cuDNN autotuning, allocator warm-up, first momentum step
            for _ in range(warmup_iters):
                self.train_step(self.static_batch)
        torch.cuda.current_stream(self.step.device).wait_stream(side)
        torch.cuda.synchronize(self.step.device)
        self._record_graph()

    def _record_graph(self) -> None:
        self.graph = torch.cuda.CUDAGraph()
        self.graph_lr = self.wl.lr(self.iteration)
        with torch.cuda.graph(self.graph):
            self.static_loss = self.forward_backward(self.static_batch)
            self.step._enqueue_device_step(self.graph_lr, torch.cuda.current_stream(self.step.device))

    def replay_step(self) -> torch.Tensor:
        """One iteration by graph replay; returns the (static) loss tensor."""
        lr = self.wl.lr(self.iteration)
        if lr != self.graph_lr:
            torch.cuda.synchronize(self.step.device)
            self._record_graph()
        ev = self._begin()
        self.graph.replay()
        self.step._log_step(lr)
        self._end(ev, self.static_loss)
        self.iteration += 1
        return self.static_loss

    # ------------------------------------------------------------------ trace
    def metrics_rows(self) -> list[dict]:
        """The iterations still in the trace ring as reference MetricsRecord
        rows (metrics.py:23-48) with loss and step_duration filled."""
        from . import trace as T

        self.step.synchronize()
        cap = self._loss_ring.numel()
        losses_dev = self._loss_ring.cpu().tolist()
        losses, durations = {}, {}
        for it, (a, b) in self._events.items():
            losses[it] = losses_dev[it % cap]
            durations[it] = a.elapsed_time(b) / 1e3  # seconds, like time.monotonic() deltas
        n_params = self.flat.n_real
        return T.to_metrics_rows(self.step.records(), n_params=n_params, losses=losses,
                                 durations=durations)
