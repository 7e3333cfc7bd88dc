"""CPU oracle for the SelSync selective-synchronization hot path.

TEST INFRASTRUCTURE ONLY. Nothing in the product package imports this module:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` arm may use it, and only as the checker or the timed CPU
reference -- never as the thing measured on the GPU path.

It is a float64 numpy restatement of the reference package (``selsync``, pure
Python + numpy, /root/reference/pkg/src/selsync) for exactly the functions on
the hot path. Each function cites the reference file:line it follows. Parity
of this restatement with the reference itself is pinned by
``tests/golden/*.npz``, which ``tests/golden/make_golden.py`` produced by
running the *unmodified* reference ``run_simulation`` (see
``tests/test_oracle_golden.py``).

Third-party arithmetic the reference delegates to: numpy 2.3.5 / OpenBLAS
0.3.30 (``ndarray @`` for the squared norm, ``np.stack(...).mean(axis=0)`` for
the parameter mean). Both are called the same way here, so the restatement is
bit-identical to the reference on the same inputs.

Momentum / weight decay are NOT in the reference (plain SGD only,
SPEC.md:109). ``sgd_momentum_step`` restates ``torch.optim.SGD``'s published
update rule (PyTorch docs, "SGD" algorithm box; torch/optim/sgd.py
``_single_tensor_sgd``) in float64; with momentum=weight_decay=0 it reduces to
the reference ``sgd_step``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, Optional

import numpy as np


class OracleSignalError(ValueError):
    """Mirror of selsync.errors.SignalError (errors.py:8-9)."""


class OracleConfigError(ValueError):
    """Mirror of selsync.errors.ConfigError (errors.py:4-5)."""


# ---------------------------------------------------------------------------
# L1 signal: signal.py:20-124


def default_smoothing(n_workers: int) -> float:
    """signal.py:20-29 -- lambda = clamp(N/100, 0.01, 1), N=1 -> 0.05."""
    if n_workers < 1:
        raise OracleConfigError(f"n_workers must be positive, got {n_workers}")
    if n_workers == 1:
        return 0.05
    return float(min(1.0, max(0.01, n_workers / 100.0)))


@dataclass(frozen=True)
class SignalState:
    """signal.py:41-61 (GradSignalState)."""

    smoothing: float
    warmup: int = 25
    ewma_current: float = 0.0
    ewma_previous: float = 0.0
    step_count: int = 0
    max_delta_seen: float = 0.0

    def __post_init__(self):
        if not (0.0 < self.smoothing <= 1.0):
            raise OracleSignalError(f"smoothing must be in (0, 1], got {self.smoothing}")
        if self.warmup < 1:
            raise OracleSignalError(f"warmup must be >= 1, got {self.warmup}")


def observe(state: SignalState, grad_norm_sq: float) -> SignalState:
    """signal.py:64-83 -- fold one squared norm into the EWMA pair."""
    x = float(grad_norm_sq)
    if np.isnan(x):
        raise OracleSignalError("observed a NaN gradient norm")
    if x < 0.0:
        raise OracleSignalError(f"squared norm cannot be negative, got {x}")
    if state.step_count == 0:
        cur = x
    else:
        cur = state.smoothing * x + (1.0 - state.smoothing) * state.ewma_current
    out = replace(state, ewma_previous=state.ewma_current, ewma_current=cur,
                  step_count=state.step_count + 1)
    if out.step_count >= 2 and out.step_count > out.warmup:
        out = replace(out, max_delta_seen=max(out.max_delta_seen, relative_change(out)))
    return out


def relative_change(state: SignalState) -> float:
    """signal.py:86-98 -- |cur-prev|/prev; 0/0 -> 0, x/0 -> inf."""
    if state.step_count < 2:
        raise OracleSignalError("relative change needs at least two observations")
    prev, cur = state.ewma_previous, state.ewma_current
    if prev == 0.0:
        return 0.0 if cur == 0.0 else float("inf")
    return abs((cur - prev) / prev)


def decide(state: SignalState, delta: float) -> str:
    """signal.py:101-107 + DeltaThreshold signal.py:32-38 (inclusive test)."""
    if not np.isfinite(delta) or delta < 0.0:
        raise OracleSignalError(f"delta must be finite and >= 0, got {delta}")
    if state.step_count < 1:
        raise OracleSignalError("decide called before any observation")
    if state.step_count <= state.warmup:
        return "sync"
    return "sync" if relative_change(state) >= delta else "local"


def replay_decisions(deltas, warmup: int, delta: float) -> int:
    """signal.py:110-124."""
    if warmup < 1:
        raise OracleConfigError(f"warmup must be >= 1, got {warmup}")
    syncs = 0
    for i, d in enumerate(deltas):
        if i < warmup or (d is not None and d >= delta):
            syncs += 1
    return syncs


# ---------------------------------------------------------------------------
# L0 numeric core: model.py:215-258


def norm_sq(grad: np.ndarray) -> float:
    """strategies.py:285 -- float(grad @ grad) in float64."""
    g = np.asarray(grad, dtype=np.float64)
    return float(g @ g)


def sgd_step(params: np.ndarray, grad: np.ndarray, lr: float) -> np.ndarray:
    """model.py:215-221 -- w - lr*g as a new array."""
    if grad.shape != params.shape:
        raise OracleConfigError("gradient shape does not match parameter vector")
    if lr < 0.0:
        raise OracleConfigError(f"learning rate must be non-negative, got {lr}")
    return params - lr * grad


def sgd_momentum_step(params, grad, buf, lr, momentum=0.0, dampening=0.0,
                      weight_decay=0.0, nesterov=False, first=False):
    """torch.optim.SGD update rule in float64 (extension; not in the reference).

    Returns (new_params, new_buf). With momentum == weight_decay == 0 this is
    exactly ``sgd_step`` (model.py:221).
    """
    d = grad
    if weight_decay != 0.0:
        d = d + weight_decay * params
    new_buf = buf
    if momentum != 0.0:
        if first or buf is None:
            new_buf = d.copy()
        else:
            new_buf = momentum * buf + (1.0 - dampening) * d
        d = d + momentum * new_buf if nesterov else new_buf
    return params - lr * d, new_buf


@dataclass(frozen=True)
class LrSchedule:
    """model.py:224-249."""

    initial_lr: float
    milestones: tuple = ()
    mode: str = "per_step"


def lr_at(schedule: LrSchedule, step: int, epoch: int) -> float:
    """model.py:252-258."""
    pos = step if schedule.mode == "per_step" else epoch
    lr = schedule.initial_lr
    for boundary, factor in schedule.milestones:
        if boundary <= pos:
            lr *= factor
    return lr


# ---------------------------------------------------------------------------
# L3/L5 aggregation and flags


def aggregate_mean(vectors: list[np.ndarray]) -> np.ndarray:
    """strategies.py:159-168 -- np.stack(...).mean(axis=0) in the given order."""
    if not vectors:
        raise ValueError("aggregate_mean needs at least one vector")
    return np.stack(vectors).mean(axis=0)


def flag_word(n_workers: int, set_ids) -> bytes:
    """wire.py:130-136 -- ceil(N/8) bytes, LSB-first."""
    word = bytearray((n_workers + 7) // 8)
    for i in set_ids:
        if not (0 <= i < n_workers):
            raise ValueError(f"flag bit {i} out of range for {n_workers} workers")
        word[i // 8] |= 1 << (i % 8)
    return bytes(word)


def or_words(words, n_workers: int) -> bytes:
    """wire.py:139-147 -- the PS OR of runtime.py:329-333."""
    out = bytearray((n_workers + 7) // 8)
    for w in words:
        for i, b in enumerate(w):
            out[i] |= b
    return bytes(out)


def any_flag(word: bytes) -> bool:
    """wire.py:150-151."""
    return any(word)


# ---------------------------------------------------------------------------
# Synthetic inputs shared by the golden generator, the tests and bench.py


def grad_scale(step: int, worker: int) -> float:
    """s = 1 + 0.6 sin(step/5) + 0.1 rank."""
    return 1.0 + 0.6 * math.sin(step / 5.0) + 0.1 * worker


def synthetic_grad32(seed: int, worker: int, step: int, n: int) -> np.ndarray:
    """fp32 gradient g[worker, step] = s(step, worker) * N(0, 1), seeded by
    SeedSequence([seed, worker, step]). Both sides consume these exact fp32
    values (the oracle upcasts them to float64)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, worker, step]))
    z = rng.standard_normal(n, dtype=np.float32)
    return z * np.float32(grad_scale(step, worker))


# ---------------------------------------------------------------------------
# N-worker lockstep restatement of _selsync_step + the parameter server


@dataclass
class SimResult:
    grad_norm_sq: np.ndarray  # (steps, N)
    ewma: np.ndarray  # (steps, N)
    delta_g: np.ndarray  # (steps, N); NaN where the reference records None
    votes: np.ndarray  # (steps, N) bool, each worker's own decide() == "sync"
    decision: np.ndarray  # (steps,) bool, True = sync (OR of votes)
    finals: np.ndarray  # (N, P)
    trajectory: dict = field(default_factory=dict)  # step -> (N, P)
    states: list = field(default_factory=list)  # final SignalState per worker


def simulate_selsync(
    init_params: np.ndarray,
    n_workers: int,
    steps: int,
    grad_fn: Callable[[int, int, np.ndarray], np.ndarray],
    *,
    delta: float,
    warmup: int = 25,
    smoothing: Optional[float] = None,
    lr: float | Callable[[int], float] = 0.1,
    aggregation: str = "params",
    momentum: float = 0.0,
    dampening: float = 0.0,
    weight_decay: float = 0.0,
    nesterov: bool = False,
    capture: Optional[Callable[[int], bool]] = None,
) -> SimResult:
    """Lockstep SelSync over N workers, float64.

    Per step and worker, in the order of strategies.py:369-403:
      grad = grad_fn(worker, step, params)        (forward_backward, :378)
      gnorm2 = grad @ grad; observe; relative_change when step_count >= 2
                                                  (_grad_and_signal, :283-288)
      PA: params = sgd_step(params, grad, lr)     (:380-383, local update first)
      own vote = decide(...) == "sync"            (:384)
    then the PS ORs all N flag words (runtime.py:319-333) and, when any bit
    is set, averages the pushed vectors in sorted worker order
    (runtime.py:275-294 -> aggregate_mean strategies.py:159-168). Under GA the
    mean gradient is applied instead (:395-397) and a local step applies the
    own gradient after the vote (:398-399). The schedule interleaving cannot
    change lockstep math (test_runtime.py:209-219), so none is modelled.
    """
    if aggregation not in ("params", "grads"):
        raise OracleConfigError(f"aggregation must be params or grads, got {aggregation!r}")
    lam = default_smoothing(n_workers) if smoothing is None else smoothing
    lr_fn = lr if callable(lr) else (lambda _s, _v=float(lr): _v)
    params = [np.array(init_params, dtype=np.float64, copy=True) for _ in range(n_workers)]
    bufs = [None] * n_workers
    states = [SignalState(smoothing=lam, warmup=warmup) for _ in range(n_workers)]
    out_g = np.zeros((steps, n_workers))
    out_e = np.zeros((steps, n_workers))
    out_d = np.full((steps, n_workers), np.nan)
    out_v = np.zeros((steps, n_workers), dtype=bool)
    out_dec = np.zeros(steps, dtype=bool)
    traj = {}
    for step in range(steps):
        lr_s = lr_fn(step)
        grads = []
        for w in range(n_workers):
            g = np.asarray(grad_fn(w, step, params[w]), dtype=np.float64)
            grads.append(g)
            gn = norm_sq(g)
            states[w] = observe(states[w], gn)
            out_g[step, w] = gn
            out_e[step, w] = states[w].ewma_current
            if states[w].step_count >= 2:
                out_d[step, w] = relative_change(states[w])
            if aggregation == "params":
                params[w], bufs[w] = sgd_momentum_step(
                    params[w], g, bufs[w], lr_s, momentum, dampening, weight_decay,
                    nesterov, first=(step == 0))
            out_v[step, w] = decide(states[w], delta) == "sync"
        words = [flag_word(n_workers, {w} if out_v[step, w] else set())
                 for w in range(n_workers)]
        synced = any_flag(or_words(words, n_workers))
        out_dec[step] = synced
        if synced:
            if aggregation == "params":
                mean = aggregate_mean([params[w] for w in range(n_workers)])
                params = [mean.copy() for _ in range(n_workers)]
            else:
                mean_g = aggregate_mean(grads)
                for w in range(n_workers):
                    params[w], bufs[w] = sgd_momentum_step(
                        params[w], mean_g, bufs[w], lr_s, momentum, dampening,
                        weight_decay, nesterov, first=(step == 0))
        elif aggregation == "grads":
            for w in range(n_workers):
                params[w], bufs[w] = sgd_momentum_step(
                    params[w], grads[w], bufs[w], lr_s, momentum, dampening,
                    weight_decay, nesterov, first=(step == 0))
        if capture is not None and capture(step):
            traj[step] = np.stack(params)
    return SimResult(out_g, out_e, out_d, out_v, out_dec, np.stack(params), traj, states)


def init_params_linear(d: int, seed: int) -> np.ndarray:
    """model.py:89-100 for ModelSpec(d, (), 2, init_seed=seed): weights
    U(-1/sqrt(d), 1/sqrt(d)) of shape (d, 2) then 2 zero biases; P = 2d + 2."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(d)
    w = rng.uniform(-bound, bound, size=(d, 2))
    out = np.zeros(2 * d + 2)
    out[: 2 * d] = w.ravel()
    return out
