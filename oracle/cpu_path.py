"""The reference's CPU work for one SelSync step, for timing only.

TEST/BENCH INFRASTRUCTURE: used solely by ``bench.py``'s ``cpu_baseline``
leg and its ``--impl reference`` arm. It restates, in the reference's own
float64 numpy operations and data movement, what one lockstep SelSync step
costs the reference for N workers + its parameter server
(``_selsync_step`` strategies.py:369-403 with the server's ``_on_flags``
runtime.py:319-333 and ``_close_round`` runtime.py:275-294):

  per worker   g @ g (:285); observe/relative_change/decide (signal.py:64-107);
               the local update (sgd_step model.py:215-221, here with the
               torch.optim.SGD momentum/weight-decay rule the GPU arm runs);
               flag_word (wire.py:130-136)
  server       or_words over the N flag words (wire.py:139-147)
  sync steps   vector_to_bytes of every worker's params (wire.py:113-114),
               bytes_to_vector at the server, np.stack(...).mean(axis=0)
               (strategies.py:159-168), one vector_to_bytes of the mean, and
               bytes_to_vector on every worker (wire.py:117-123)

Workers run concurrently on a thread pool (numpy releases the GIL on these
array operations), so the baseline uses up to ``threads`` host cores.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import selsync_oracle as O


class CpuSelSync:
    def __init__(self, n_workers: int, P: int, *, delta: float, warmup: int, smoothing: float,
                 momentum: float, weight_decay: float, grad_ring: int = 4, sync_pattern=None,
                 threads: int | None = None, seed: int = 0):
        self.n, self.P = n_workers, P
        self.delta, self.momentum, self.wd = delta, momentum, weight_decay
        rng = np.random.default_rng(seed)
        init = rng.uniform(-0.05, 0.05, size=P)
        self.params = [init.copy() for _ in range(n_workers)]
        self.bufs = [None] * n_workers
        self.states = [O.SignalState(smoothing=smoothing, warmup=warmup) for _ in range(n_workers)]
        scales = sync_pattern or [1.0] * grad_ring
        base = [rng.standard_normal(P) for _ in range(min(grad_ring, 2))]
        self.ring = [[base[(k + w) % len(base)] * scales[k % len(scales)] for k in range(grad_ring)]
                     for w in range(n_workers)]
        self.threads = max(1, min(threads or os.cpu_count() or 1, n_workers))
        self.pool = ThreadPoolExecutor(self.threads)
        self.step_idx = 0
        self.syncs = 0

    def _worker(self, w: int, lr: float) -> bool:
        g = self.ring[w][self.step_idx % len(self.ring[w])]
        gn = float(g @ g)
        self.states[w] = O.observe(self.states[w], gn)
        if self.states[w].step_count >= 2:
            O.relative_change(self.states[w])
        self.params[w], self.bufs[w] = O.sgd_momentum_step(
            self.params[w], g, self.bufs[w], lr, self.momentum, 0.0, self.wd, False,
            first=(self.step_idx == 0))
        return O.decide(self.states[w], self.delta) == "sync"

    def step(self, lr: float) -> bool:
        votes = list(self.pool.map(lambda w: self._worker(w, lr), range(self.n)))
        words = [O.flag_word(self.n, {w} if v else set()) for w, v in enumerate(votes)]
        synced = O.any_flag(O.or_words(words, self.n))
        if synced:
            pushed = list(self.pool.map(lambda w: np.ascontiguousarray(self.params[w], dtype="<f8").tobytes(),
                                        range(self.n)))
            vecs = list(self.pool.map(lambda b: np.frombuffer(b, dtype="<f8").astype(np.float64), pushed))
            mean = O.aggregate_mean(vecs)
            payload = np.ascontiguousarray(mean, dtype="<f8").tobytes()
            self.params = list(self.pool.map(
                lambda _w: np.frombuffer(payload, dtype="<f8").astype(np.float64), range(self.n)))
            self.syncs += 1
        self.step_idx += 1
        return synced

    def time_steps(self, steps: int, lr: float = 0.1) -> float:
        """Wall seconds for `steps` steps."""
        t0 = time.perf_counter()
        for _ in range(steps):
            self.step(lr)
        return time.perf_counter() - t0

    def close(self):
        self.pool.shutdown(wait=True)
