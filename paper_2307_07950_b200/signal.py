"""Scalar gradient-change detector API (reference: signal.py:20-124).

Same names, signatures, value semantics and exceptions as the reference's
``selsync.signal``. The arithmetic is NOT re-implemented here: every call goes
through the native host entry points of libselsync_b200.so
(``ss_signal_observe`` / ``ss_relative_change`` / ``ss_decide``), which share
one ``__host__ __device__`` implementation with the on-device signal step K2.
So the scalar API, the device kernel and the reference round identically
(one IEEE rounding per Python float operation, no FMA contraction).

The per-step device path lives in :mod:`paper_2307_07950_b200.step`; this
module is for host-side inspection, replay and tests.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from . import _native as N
from .errors import ConfigError, SignalError


def default_smoothing(n_workers: int) -> float:
    """lambda = clamp(N/100, 0.01, 1.0); a single worker gets 0.05 (signal.py:20-29)."""
    out = ctypes.c_double(0.0)
    N.check(N.LIB.ss_default_smoothing(int(n_workers), ctypes.byref(out)))
    return float(out.value)


@dataclass(frozen=True)
class DeltaThreshold:
    """delta >= 0 and finite (signal.py:32-38)."""

    delta: float

    def __post_init__(self):
        N.check(N.LIB.ss_check_delta(float(self.delta)))


@dataclass(frozen=True)
class GradSignalState:
    """EWMA pair over observed squared gradient norms (signal.py:41-61)."""

    smoothing: float
    warmup: int = 25
    ewma_current: float = 0.0
    ewma_previous: float = 0.0
    step_count: int = 0
    max_delta_seen: float = 0.0

    def __post_init__(self):
        if not (0.0 < self.smoothing <= 1.0):
            raise SignalError(f"smoothing must be in (0, 1], got {self.smoothing}")
        if self.warmup < 1:
            raise SignalError(f"warmup must be >= 1, got {self.warmup}")

    # -- native struct conversion ------------------------------------------
    def to_c(self) -> N.SignalStateC:
        c = N.SignalStateC()
        c.smoothing = self.smoothing
        c.warmup = self.warmup
        c.ewma_current = self.ewma_current
        c.ewma_previous = self.ewma_previous
        c.step_count = self.step_count
        c.max_delta_seen = self.max_delta_seen
        c.last_delta = math.nan
        c.error = 0
        return c

    @classmethod
    def from_c(cls, c: N.SignalStateC) -> "GradSignalState":
        return cls(
            smoothing=c.smoothing,
            warmup=c.warmup,
            ewma_current=c.ewma_current,
            ewma_previous=c.ewma_previous,
            step_count=c.step_count,
            max_delta_seen=c.max_delta_seen,
        )


def observe(state: GradSignalState, grad_norm_sq: float) -> GradSignalState:
    """Fold one squared gradient norm into the EWMA pair; returns the new state
    (signal.py:64-83). NaN / negative raise SignalError; the input state is
    never modified."""
    c = state.to_c()
    N.check(N.LIB.ss_signal_observe(ctypes.byref(c), float(grad_norm_sq)))
    return GradSignalState.from_c(c)


def relative_change(state: GradSignalState) -> float:
    """|ewma_current - ewma_previous| / ewma_previous; 0/0 -> 0, x/0 -> inf
    (signal.py:86-98)."""
    c = state.to_c()
    out = ctypes.c_double(0.0)
    N.check(N.LIB.ss_relative_change(ctypes.byref(c), ctypes.byref(out)))
    return float(out.value)


def decide(state: GradSignalState, threshold: DeltaThreshold) -> str:
    """'sync' or 'local'; warmup steps always sync, the test is inclusive
    (signal.py:101-107)."""
    c = state.to_c()
    out = ctypes.c_int32(0)
    N.check(N.LIB.ss_decide(ctypes.byref(c), float(threshold.delta), ctypes.byref(out)))
    return "sync" if out.value else "local"


def sync_known_ahead(state: GradSignalState, threshold: DeltaThreshold) -> bool:
    """True when the decision after the next observation is "sync" whatever
    the observed norm: a warmup step, or delta == 0. Not in the reference; the
    one-launch step uses the same predicate to start the mean before ||g||^2
    is known (known-sync pass)."""
    c = state.to_c()
    out = ctypes.c_int32(0)
    N.check(N.LIB.ss_sync_known_ahead(ctypes.byref(c), float(threshold.delta), ctypes.byref(out)))
    return bool(out.value)


def sync_proven_early(state: GradSignalState, threshold: DeltaThreshold, lower: float) -> bool:
    """True when observing ANY norm >= ``lower`` next is proven to decide
    "sync" on the upward side (new EWMA >= previous): the exact early vote the
    norm-first step posts from a running partial sum of ||g||^2 before the
    sweep ends. Sound, not complete. Not in the reference (it restates
    signal.py:64-107 over an interval)."""
    c = state.to_c()
    out = ctypes.c_int32(0)
    N.check(N.LIB.ss_sync_proven_early(ctypes.byref(c), float(lower), float(threshold.delta), ctypes.byref(out)))
    return bool(out.value)


def replay_decisions(deltas, warmup: int, delta: float) -> int:
    """Count sync decisions of a recorded Delta trace at one threshold
    (signal.py:110-124); entries recorded during warmup are None."""
    if warmup < 1:
        raise ConfigError(f"warmup must be >= 1, got {warmup}")
    return sum(1 for i, d in enumerate(deltas) if i < warmup or (d is not None and d >= delta))


__all__ = [
    "DeltaThreshold",
    "GradSignalState",
    "decide",
    "default_smoothing",
    "observe",
    "relative_change",
    "replay_decisions",
    "sync_known_ahead",
]
