"""B200-native SelSync hot path (arXiv 2307.07950), drop-in for the reference's
step/decision interface.

Reference API kept (same names and semantics, /root/reference/pkg/src/selsync):
  signal:  default_smoothing, DeltaThreshold, GradSignalState, observe,
           relative_change, decide, replay_decisions
  config:  SelSyncConfig (delta, aggregation, warmup, smoothing [+ momentum,
           dampening, weight_decay, nesterov])
  model:   ParamVector, sgd_step, aggregate_mean, LrSchedule, lr_at
  data:    split_chunks, plan_defdp, plan_seldp, bind_plan, ChunkSampler (SelDP)
  wire:    flag_word, or_words, any_flag (flag semantics)
  errors:  ConfigError, SignalError, ProtocolError, TransportError
New:
  sync_known_ahead  the decision after the next observation is sync whatever
                    the norm (warmup, delta == 0): the known-sync pass
  SelSyncStep     one rank's step over flat fp32 buffers (NCCL across GPUs)
  ReplicaSelSync  N simulated workers on one GPU
  FlatParameters  p.data / p.grad as views of flat buffers
"""

from .errors import ConfigError, ProtocolError, SignalError, TransportError  # noqa: F401
from . import _native  # noqa: F401  (loads libselsync_b200.so; raises if missing)
from .signal import (  # noqa: F401
    DeltaThreshold,
    GradSignalState,
    decide,
    default_smoothing,
    observe,
    relative_change,
    replay_decisions,
    sync_known_ahead,
)
from .config import AGG_MODES, SelSyncConfig  # noqa: F401
from .data import (  # noqa: F401
    ChunkSampler,
    ChunkSplit,
    PartitionPlan,
    TokenStreamSampler,
    bind_plan,
    plan_call_count,
    plan_defdp,
    plan_seldp,
    split_chunks,
)
from .wire import any_flag, flag_word, flag_word_size, flags_in_word, or_words  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent parts load lazily so the scalar API imports fast
    if name in ("SelSyncStep", "TensorListSelSyncStep"):
        from . import step
        return getattr(step, name)
    if name in ("SelSyncTrainer",):
        from .train import SelSyncTrainer
        return SelSyncTrainer
    if name in ("ReplicaSelSync",):
        from .replicas import ReplicaSelSync
        return ReplicaSelSync
    if name in ("FlatParameters", "ParamVector", "sgd_step", "aggregate_mean", "LrSchedule",
                "lr_at", "flat_layout"):
        from . import model
        return getattr(model, name)
    if name in ("RankGroup",):
        from .collectives import RankGroup
        return RankGroup
    raise AttributeError(name)
