"""N simulated SelSync workers on one device.

The device counterpart of the reference's in-process cluster
(``run_simulation``, runtime.py:462-581): N replicas of the flat parameter
buffer, each with its own device signal state, stepped in lockstep. The
exchanges that NCCL performs across GPUs in :class:`SelSyncStep` are device
kernels here: ``ss_replica_flag_max_i32`` (the PS flag OR, runtime.py:319-333)
and ``ss_replica_average_f32`` (the PS mean in sorted worker order,
runtime.py:275-294 -> strategies.py:159-168). Used for BASELINE config 0
("2 simulated workers") and for N-worker decision-trace parity on one GPU.
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import torch

from . import kernels as K
from .config import SelSyncConfig
from .errors import ConfigError


class ReplicaSelSync:
    def __init__(self, init_params: torch.Tensor, n_workers: int, config: SelSyncConfig, *,
                 fuse: bool = True, trace_capacity: int = 4096):
        K._need(init_params, torch.float32, "init_params")
        if n_workers < 1 or n_workers > 64:
            raise ConfigError(f"n_workers must be in [1, 64], got {n_workers}")
        self.config = config
        self.n = n_workers
        self.device = init_params.device
        self.fuse = bool(fuse) and config.aggregation == "params"
        p = init_params.reshape(-1)
        # bootstrap: every replica pulls the same initial vector (runtime.py:178-191)
        self.params = [p.clone() for _ in range(n_workers)]
        self.grads = [torch.zeros_like(p) for _ in range(n_workers)]
        self.moms = ([torch.zeros_like(p) for _ in range(n_workers)]
                     if config.momentum != 0.0 else [None] * n_workers)
        lam = config.smoothing_for(n_workers)
        self.signals = [K.DeviceSignal(self.device, lam, config.warmup, trace_capacity)
                        for _ in range(n_workers)]
        self.ws = K.Workspace(self.device)  # kernels serialise on one stream
        self._word_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._ready = torch.cuda.Event()
        self.steps_done = 0
        self.decisions: list[bool] = []

    def set_grads(self, grads: Sequence[torch.Tensor]) -> None:
        for dst, src in zip(self.grads, grads):
            dst.copy_(src.reshape(-1), non_blocking=True)

    def step(self, lr: float) -> str:
        cfg = self.config
        first = self.steps_done == 0
        hp = dict(momentum=cfg.momentum, dampening=cfg.dampening, weight_decay=cfg.weight_decay,
                  nesterov=cfg.nesterov, first_step=first)
        for r in range(self.n):
            if self.fuse:
                K.update_norm_signal_(self.params[r], self.grads[r], self.moms[r], self.signals[r],
                                      self.ws, lr=lr, delta=cfg.delta, **hp)
            else:
                K.norm_signal(self.grads[r], self.signals[r], cfg.delta, self.ws)
        words = [s.word for s in self.signals]
        K.replica_flag_max_(words)
        if cfg.aggregation == "params" and not self.fuse:
            for r in range(self.n):
                K.sgd_update_(self.params[r], self.grads[r], self.moms[r], lr=lr,
                              sync_word=words[r], sync_scale=1.0 / self.n, **hp)
        self._word_host.copy_(words[0], non_blocking=True)
        self._ready.record(torch.cuda.current_stream(self.device))
        self._ready.synchronize()
        word = int(self._word_host[0])
        if word >= 2:
            K.raise_for_word(word, f" at step {self.steps_done}")
        synced = bool(word & 1)
        if cfg.aggregation == "params":
            if synced:
                if self.fuse:
                    K.replica_average_(self.params)
                else:  # pre-scaled by 1/N in the update epilogue: the sum is the mean
                    K.replica_average_(self.params, divide=False)
        else:
            if synced:
                K.replica_average_(self.grads)
            for r in range(self.n):
                K.sgd_update_(self.params[r], self.grads[r], self.moms[r], lr=lr, **hp)
        self.steps_done += 1
        self.decisions.append(synced)
        return "sync" if synced else "local"

    def trace(self, worker: int):
        return self.signals[worker].read_trace()

    def records(self) -> list[dict]:
        out = []
        for w in range(self.n):
            rows = self.signals[w].read_trace()
            cap = self.signals[w].trace_capacity
            for step in range(max(0, self.steps_done - cap), self.steps_done):
                r = rows[step % cap]
                d = float(r["delta_g"])
                out.append(dict(step=step, worker_id=w, grad_norm_sq=float(r["grad_norm_sq"]),
                                ewma=float(r["ewma"]), delta_g=None if math.isnan(d) else d,
                                decision="sync" if self.decisions[step] else "local",
                                vote=bool(int(r["word"]) & 1)))
        return out
