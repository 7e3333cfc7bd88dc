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
    def __init__(self, workload: Workload, *, delta: float, warmup: int = 25,
                 smoothing: Optional[float] = None, group=None, **step_kw):
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
        loss = self.forward_backward(batch)
        lr = self.wl.lr(self.iteration)
        if wait or not self.step.async_capable:
            decision = self.step.step(lr)
        else:
            self.step.step_async(lr)
            decision = None
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
        self.graph.replay()
        self.step._log_step(lr)
        self.iteration += 1
        return self.static_loss
