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
