"""SelSync configuration (reference: strategies.py:56-61, :106-121; JSON keys
experiment.py:189-196).

``delta``, ``aggregation``, ``warmup`` and ``smoothing`` keep the reference's
names, defaults and validation. The optimizer fields are the B200 build's
extension (the reference is plain SGD): with their defaults the
update is exactly ``sgd_step`` (model.py:215-221).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass
from typing import Optional

from .errors import ConfigError
from .signal import DeltaThreshold, default_smoothing

AGG_MODES = ("params", "grads")


def _check_agg(mode: str) -> None:
    if mode not in AGG_MODES:
        raise ConfigError(f"aggregation must be one of {AGG_MODES}, got {mode!r}")


@dataclass(frozen=True)
class SelSyncConfig:
    """Synchronize a step only when any worker's gradient signal crosses delta."""

    delta: float
    aggregation: str = "params"
    warmup: int = 25
    smoothing: Optional[float] = None
    # --- B200 extension: torch.optim.SGD-style local update
    momentum: float = 0.0
    dampening: float = 0.0
    weight_decay: float = 0.0
    nesterov: bool = False

    def __post_init__(self):
        _check_agg(self.aggregation)
        DeltaThreshold(self.delta)  # range check, signal.py:36-38
        if self.warmup < 1:
            raise ConfigError(f"warmup must be >= 1, got {self.warmup}")
        if self.smoothing is not None and not 0.0 < self.smoothing <= 1.0:
            raise ConfigError(f"smoothing must be in (0, 1], got {self.smoothing}")
        for name in ("momentum", "dampening", "weight_decay"):
            v = getattr(self, name)
            if not math.isfinite(v) or v < 0.0:
                raise ConfigError(f"{name} must be finite and >= 0, got {v}")
        if self.nesterov and (self.momentum <= 0.0 or self.dampening != 0.0):
            raise ConfigError("Nesterov momentum requires a momentum and zero dampening")

    def smoothing_for(self, n_workers: int) -> float:
        """strategies.py:206-213: an unset smoothing resolves to default_smoothing(N)."""
        return default_smoothing(n_workers) if self.smoothing is None else float(self.smoothing)

    def to_json(self) -> dict:
        return {"kind": "selsync", **asdict(self)}

    @classmethod
    def from_json(cls, obj: dict) -> "SelSyncConfig":
        """Accepts the reference's strategy object (experiment.py:189-196)."""
        if obj.get("kind", "selsync") != "selsync":
            raise ConfigError(f"not a selsync strategy: {obj.get('kind')!r}")
        if "delta" not in obj:
            raise ConfigError("selsync strategy needs 'delta'")
        keys = ("delta", "aggregation", "warmup", "smoothing", "momentum", "dampening",
                "weight_decay", "nesterov")
        return cls(**{k: obj[k] for k in keys if k in obj})
