"""Flat parameter vectors on the device (reference: model.py:54-82, :215-258;
strategies.py:159-168).

``ParamVector`` keeps the reference's (values, layout) shape, but ``values``
is a flat fp32 CUDA tensor and the layout offsets are padded to 16-byte
boundaries so every tensor view -- and the whole buffer -- streams with
128-bit accesses. ``sgd_step`` and ``aggregate_mean`` keep value semantics
(fresh output, inputs untouched) and run on the sm_100a kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod
from typing import Iterable, Sequence

import torch

from . import kernels as K
from .errors import ConfigError

ALIGN_ELEMS = 4  # 16 bytes of fp32


def _pad(n: int) -> int:
    return (n + ALIGN_ELEMS - 1) // ALIGN_ELEMS * ALIGN_ELEMS


def flat_layout(shapes: Iterable[Sequence[int]]) -> tuple[tuple[tuple[int, tuple[int, ...]], ...], int]:
    """(offset, shape) per tensor (model.py:74-82), offsets 16-byte aligned; returns (layout, P_padded)."""
    layout = []
    off = 0
    for shape in shapes:
        shape = tuple(int(s) for s in shape)
        layout.append((off, shape))
        off += _pad(prod(shape))
    return tuple(layout), off


@dataclass
class ParamVector:
    """Flat fp32 device vector plus (offset, shape) layout per tensor (model.py:54-66)."""

    values: torch.Tensor
    layout: tuple

    def copy(self) -> "ParamVector":
        return ParamVector(self.values.clone(), self.layout)

    def tensor(self, i: int) -> torch.Tensor:
        off, shape = self.layout[i]
        return self.values[off: off + prod(shape)].view(shape)


def sgd_step(params: ParamVector, grad: torch.Tensor, lr: float) -> ParamVector:
    """w - lr * g as a new vector; the input is left unmodified (model.py:215-221)."""
    if grad.shape != params.values.shape:
        raise ConfigError("gradient shape does not match parameter vector")
    if lr < 0.0:
        raise ConfigError(f"learning rate must be non-negative, got {lr}")
    out = params.values.clone()
    K.sgd_update_(out, grad, None, lr=lr)
    return ParamVector(out, params.layout)


def aggregate_mean(vectors: list[ParamVector]) -> ParamVector:
    """Elementwise arithmetic mean of identically laid out vectors (strategies.py:159-168)."""
    if not vectors:
        raise ValueError("aggregate_mean needs at least one vector")
    layout = vectors[0].layout
    for v in vectors[1:]:
        if v.layout != layout:
            raise ValueError("aggregate_mean: layout mismatch")
    return ParamVector(K.mean([v.values for v in vectors]), layout)


@dataclass(frozen=True)
class LrSchedule:
    """Piecewise-constant decay (model.py:224-249)."""

    initial_lr: float
    milestones: tuple = ()
    mode: str = "per_step"

    def __post_init__(self):
        object.__setattr__(self, "milestones",
                           tuple((int(b), float(f)) for b, f in self.milestones))
        if self.initial_lr <= 0.0:
            raise ConfigError(f"initial_lr must be positive, got {self.initial_lr}")
        if self.mode not in ("per_step", "per_epoch"):
            raise ConfigError(f"schedule mode must be per_step or per_epoch, got {self.mode!r}")
        bounds = [b for b, _ in self.milestones]
        if any(b2 <= b1 for b1, b2 in zip(bounds, bounds[1:])):
            raise ConfigError("milestone boundaries must be strictly increasing")
        if any(f <= 0.0 for _, f in self.milestones):
            raise ConfigError("milestone factors must be positive")


def lr_at(schedule: LrSchedule, step: int, epoch: int) -> float:
    """lr = initial * prod(factor for boundary <= position) (model.py:252-258)."""
    pos = step if schedule.mode == "per_step" else epoch
    lr = schedule.initial_lr
    for boundary, factor in schedule.milestones:
        if boundary <= pos:
            lr *= factor
    return lr


class FlatParameters:
    """Flat fp32 param / grad (/ momentum) buffers behind a torch model.

    Every ``p.data`` becomes a view into ``params`` and every ``p.grad`` a
    view into ``grads``, so ``loss.backward()`` accumulates straight into the
    flat buffer and the hot path streams one contiguous allocation (no gather
    copy). Call ``zero_grad()`` (not ``optimizer.zero_grad(set_to_none=True)``)
    between steps.
    """

    def __init__(self, parameters: Iterable[torch.nn.Parameter], device=None, momentum: bool = False):
        self.parameters = [p for p in parameters if p.requires_grad]
        if not self.parameters:
            raise ConfigError("no trainable parameters")
        dev = torch.device(device) if device is not None else self.parameters[0].device
        if dev.type != "cuda":
            raise ConfigError("FlatParameters needs a CUDA device")
        self.layout, self.numel = flat_layout(p.shape for p in self.parameters)
        self.params = torch.zeros(self.numel, dtype=torch.float32, device=dev)
        self.grads = torch.zeros(self.numel, dtype=torch.float32, device=dev)
        self.momentum = torch.zeros(self.numel, dtype=torch.float32, device=dev) if momentum else None
        # 4-D tensors already in channels_last keep that layout: their views into
        # the flat buffers get NHWC strides (cuDNN then needs no weight transposes)
        self.channels_last = [p.dim() == 4 and not p.is_contiguous()
                              and p.is_contiguous(memory_format=torch.channels_last)
                              for p in self.parameters]
        with torch.no_grad():
            for p, (off, shape), cl in zip(self.parameters, self.layout, self.channels_last):
                view = self._view(self.params, off, shape, cl)
                view.copy_(p.data.to(device=dev, dtype=torch.float32))
                p.data = view
                p.grad = self._view(self.grads, off, shape, cl)

    @staticmethod
    def _view(buf: torch.Tensor, off: int, shape, channels_last: bool) -> torch.Tensor:
        flat = buf[off: off + prod(shape)]
        if channels_last:
            n, c, h, w = shape
            return flat.view(n, h, w, c).permute(0, 3, 1, 2)
        return flat.view(shape)

    @property
    def n_real(self) -> int:
        return sum(prod(s) for _, s in self.layout)

    def zero_grad(self) -> None:
        self.grads.zero_()

    def rebind(self, params: torch.Tensor) -> None:
        """Point every ``p.data`` at views of another flat buffer with the same
        layout (e.g. the symmetric-memory copy owned by a SelSyncStep)."""
        if params.numel() != self.numel or params.dtype != torch.float32:
            raise ConfigError("rebind needs a flat fp32 buffer of the same padded size")
        for p, (off, shape), cl in zip(self.parameters, self.layout, self.channels_last):
            p.data = self._view(params, off, shape, cl)
        self.params = params

    def rebind_grads(self, grads: torch.Tensor) -> None:
        """Point every ``p.grad`` at views of another flat buffer (e.g. the
        symmetric-memory gradient of a gradient-aggregation SelSyncStep)."""
        if grads.numel() != self.numel or grads.dtype != torch.float32:
            raise ConfigError("rebind_grads needs a flat fp32 buffer of the same padded size")
        for p, (off, shape), cl in zip(self.parameters, self.layout, self.channels_last):
            p.grad = self._view(grads, off, shape, cl)
        self.grads = grads

    def vector(self) -> ParamVector:
        return ParamVector(self.params, self.layout)
