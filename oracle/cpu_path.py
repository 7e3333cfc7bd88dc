"""The reference's CPU work for one SelSync step, for timing only.

TEST/BENCH INFRASTRUCTURE: used solely by ``bench.py``'s ``cpu_baseline``
leg and its ``--impl reference`` arm. It restates, in the reference's own
float64 numpy operations and data movement, what one lockstep SelSync step
costs the reference for N workers + its parameter server
(``_selsync_step`` strategies.py:369-403 with the server's ``_on_flags``
runtime.py:319-333 and ``_close_round`` runtime.py:275-294):

  per worker   g @ g (:285); observe/relative_change/decide (signal.py:64-107);
               the local update (sgd_step model.py:215-221 -- new arrays, as
               the reference allocates them -- with the torch.optim.SGD
               momentum / weight-decay rule the GPU arm runs); flag_word
               (wire.py:130-136)
  server       or_words over the N flag words (wire.py:139-147)
  sync steps   vector_to_bytes of every worker's params (wire.py:113-114),
               bytes_to_vector at the server, np.stack(...).mean(axis=0)
               (strategies.py:159-168), one vector_to_bytes of the mean, and
               bytes_to_vector on every worker (wire.py:117-123)

To use every host core, the P-long vectors are cut into as many contiguous
slices as threads and each thread runs those same numpy expressions on its
slice (numpy releases the GIL); the scalar signal step runs once per worker
on the summed slice norms.
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
        self.bufs = [np.zeros(P) for _ in range(n_workers)]
        self.states = [O.SignalState(smoothing=smoothing, warmup=warmup) for _ in range(n_workers)]
        scales = sync_pattern or [1.0] * grad_ring
        base = [rng.standard_normal(P) for _ in range(min(grad_ring, 2))]
        self.ring = [[base[(k + w) % len(base)] * scales[k % len(scales)] for k in range(grad_ring)]
                     for w in range(n_workers)]
        self.threads = max(1, threads or os.cpu_count() or 1)
        edges = np.linspace(0, P, self.threads + 1).astype(np.int64)
        self.slices = [slice(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]
        self.pool = ThreadPoolExecutor(len(self.slices))
        self.step_idx = 0
        self.syncs = 0

    def _map(self, fn):
        return list(self.pool.map(fn, self.slices))

    def step(self, lr: float) -> bool:
        k = self.step_idx % len(self.ring[0])
        grads = [self.ring[w][k] for w in range(self.n)]
        # g @ g per worker (strategies.py:285), slice partials summed
        norms = np.sum(self._map(lambda sl: [float(g[sl] @ g[sl]) for g in grads]), axis=0)
        votes = []
        for w in range(self.n):
            self.states[w] = O.observe(self.states[w], float(norms[w]))
            if self.states[w].step_count >= 2:
                O.relative_change(self.states[w])
            votes.append(O.decide(self.states[w], self.delta) == "sync")
        first = self.step_idx == 0
        mu, wd = self.momentum, self.wd

        def update(sl):  # sgd_step with momentum / weight decay, new arrays per slice
            for w in range(self.n):
                p, g, b = self.params[w][sl], grads[w][sl], self.bufs[w][sl]
                d = g + wd * p if wd else g
                if mu:
                    b = d.copy() if first else mu * b + d
                    self.bufs[w][sl] = b
                    d = b
                self.params[w][sl] = p - lr * d

        self._map(update)
        words = [O.flag_word(self.n, {w} if v else set()) for w, v in enumerate(votes)]
        synced = O.any_flag(O.or_words(words, self.n))
        if synced:
            def mean(sl):  # push (f64 bytes), PS stack + mean, pull (f64 bytes)
                pushed = [np.ascontiguousarray(self.params[w][sl], dtype="<f8").tobytes() for w in range(self.n)]
                vecs = [np.frombuffer(b, dtype="<f8").astype(np.float64) for b in pushed]
                payload = np.ascontiguousarray(np.stack(vecs).mean(axis=0), dtype="<f8").tobytes()
                for w in range(self.n):
                    self.params[w][sl] = np.frombuffer(payload, dtype="<f8").astype(np.float64)

            self._map(mean)
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
