"""SelDP partitioner and chunk samplers (reference: data.py:158-419).

Planning is a one-time host cost before training (data.py:1-6): one seeded
global shuffle cut into N near-equal contiguous chunks; DefDP gives worker i
chunk i, SelDP gives worker i the rotation i, i+1, ..., i+N-1 (mod N) per
epoch. The samplers reproduce the reference's index
streams exactly -- same numpy Generator calls, same SeedSequence keys -- so a
B200 run consumes the very batches the CPU reference would
(tests/golden/seldp_cases.npz).

The samplers only produce *indices*; ``TokenStreamSampler`` turns them into
(bptt+1)-token windows of a token stream for the Transformer-LM config, and
``indices_to_device`` stages a batch of indices for an on-device gather.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError

_plan_calls = 0


def plan_call_count() -> int:
    """How many planning routines ran in this process (data.py:27-29)."""
    return _plan_calls


def _planned() -> None:
    global _plan_calls
    _plan_calls += 1


@dataclass(frozen=True)
class ChunkSplit:
    """A fixed global shuffle cut into contiguous near-equal chunks (data.py:162-175)."""

    permutation: np.ndarray
    bounds: tuple

    def chunk_indices(self, chunk: int) -> np.ndarray:
        lo, hi = self.bounds[chunk]
        return self.permutation[lo:hi]

    @property
    def n_chunks(self) -> int:
        return len(self.bounds)


def split_chunks(n_samples: int, n_chunks: int, seed: int) -> ChunkSplit:
    """One seeded shuffle; chunk sizes differ by at most one, larger first (data.py:178-193)."""
    _planned()
    if n_chunks < 1:
        raise ConfigError(f"n_chunks must be positive, got {n_chunks}")
    if n_chunks > n_samples:
        raise ConfigError(f"cannot cut {n_samples} samples into {n_chunks} chunks")
    perm = np.random.default_rng(seed).permutation(n_samples)
    q, r = divmod(n_samples, n_chunks)
    sizes = np.full(n_chunks, q, dtype=np.int64)
    sizes[:r] += 1
    edges = np.concatenate([[0], np.cumsum(sizes)])
    return ChunkSplit(perm, tuple((int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])))


@dataclass(frozen=True)
class PartitionPlan:
    """The chunk sequence one worker traverses each epoch (data.py:196-206)."""

    worker_id: int
    chunk_order: tuple
    chunk_bounds: tuple | None = None


def _check_worker(worker_id: int, n_workers: int) -> None:
    if n_workers < 1:
        raise ConfigError(f"n_workers must be positive, got {n_workers}")
    if not (0 <= worker_id < n_workers):
        raise ConfigError(f"worker_id {worker_id} out of range for {n_workers} workers")


def bind_plan(plan: PartitionPlan, split: ChunkSplit) -> PartitionPlan:
    """Attach the split's chunk bounds (data.py:209-212)."""
    if any(c >= split.n_chunks for c in plan.chunk_order):
        raise ConfigError("plan references a chunk the split does not have")
    return PartitionPlan(plan.worker_id, plan.chunk_order, split.bounds)


def plan_defdp(worker_id: int, n_workers: int) -> PartitionPlan:
    """Default partitioning: worker i owns chunk i only (data.py:215-219)."""
    _planned()
    _check_worker(worker_id, n_workers)
    return PartitionPlan(worker_id, (worker_id,))


def plan_seldp(worker_id: int, n_workers: int) -> PartitionPlan:
    """SelDP rotation: worker i visits chunks i, i+1, ... mod N each epoch (data.py:222-226)."""
    _planned()
    _check_worker(worker_id, n_workers)
    return PartitionPlan(worker_id, tuple(int(c) for c in np.roll(np.arange(n_workers), -worker_id)))


class ChunkSampler:
    """Infinite index-batch stream over one worker's chunk traversal (data.py:364-419).

    Each epoch walks ``plan.chunk_order``; inside every chunk the order is
    reshuffled with ``SeedSequence([seed, epoch, chunk])`` (shared by all
    workers), and a tail shorter than a batch is dropped at the epoch end.
    ``next_indices`` returns (dataset indices, source chunk); ``next_batch``
    gathers rows of host arrays ``features``/``labels`` like the reference.
    """

    def __init__(self, n_samples_or_dataset, split: ChunkSplit, plan: PartitionPlan,
                 batch_size: int, seed: int):
        if batch_size < 1:
            raise ConfigError(f"batch_size must be >= 1, got {batch_size}")
        self.dataset = None if isinstance(n_samples_or_dataset, (int, np.integer)) else n_samples_or_dataset
        self.split = split
        self.plan = plan
        self.batch_size = int(batch_size)
        self.seed = seed
        self.epoch = -1
        self.pos = 0
        self._order = np.empty(0, dtype=np.int64)
        self._starts = np.zeros(1, dtype=np.int64)
        sizes = [split.bounds[c][1] - split.bounds[c][0] for c in plan.chunk_order]
        self.epoch_length = int(sum(sizes))
        if self.epoch_length < batch_size:
            raise ConfigError("worker partition smaller than one batch")

    def _new_epoch(self) -> None:
        self.epoch += 1
        pieces = []
        for c in self.plan.chunk_order:
            idx = self.split.chunk_indices(c)
            rng = np.random.default_rng(np.random.SeedSequence([self.seed, self.epoch, c]))
            pieces.append(idx[rng.permutation(idx.size)])
        self._order = np.concatenate(pieces)
        self._starts = np.cumsum([0] + [p.size for p in pieces])
        self.pos = 0

    def next_indices(self) -> tuple[np.ndarray, int]:
        if self.epoch < 0 or self.pos + self.batch_size > self._order.size:
            self._new_epoch()
        idx = self._order[self.pos: self.pos + self.batch_size]
        chunk_slot = int(np.searchsorted(self._starts, self.pos, side="right")) - 1
        self.pos += self.batch_size
        return idx, int(self.plan.chunk_order[chunk_slot])

    def next_batch(self):
        idx, source = self.next_indices()
        if self.dataset is None:
            return idx, source
        feats, labels = self.dataset
        return feats[idx], labels[idx], source


class TokenStreamSampler:
    """SelDP over a token stream (BASELINE config 3, Transformer LM).

    The stream is cut into ``n_windows`` non-overlapping windows of
    ``bptt + 1`` tokens; windows are the samples that ``split_chunks`` /
    ``plan_seldp`` partition, so the SelDP rotation and per-epoch reshuffle
    are exactly the reference's. ``next_windows`` returns the start offsets of
    one batch of windows.
    """

    def __init__(self, n_tokens: int, bptt: int, worker_id: int, n_workers: int, batch_size: int,
                 seed: int, split_seed: int = 5, scheme: str = "seldp"):
        if bptt < 1:
            raise ConfigError(f"bptt must be >= 1, got {bptt}")
        self.bptt = int(bptt)
        n_windows = (n_tokens - 1) // self.bptt
        if n_windows < n_workers:
            raise ConfigError("token stream too short for the number of workers")
        self.split = split_chunks(n_windows, n_workers, split_seed)
        planner = {"seldp": plan_seldp, "defdp": plan_defdp}.get(scheme)
        if planner is None:
            raise ConfigError(f"unknown partitioning scheme {scheme!r}")
        self.plan = bind_plan(planner(worker_id, n_workers), self.split)
        self.sampler = ChunkSampler(n_windows, self.split, self.plan, batch_size, seed)

    def next_windows(self) -> tuple[np.ndarray, int]:
        idx, source = self.sampler.next_indices()
        return idx.astype(np.int64) * self.bptt, source
