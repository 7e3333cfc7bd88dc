"""ctypes binding of ``libselsync_b200.so`` (the C-ABI in include/selsync_b200.h).

There is no Python fallback: if the shared library is missing or cannot be
loaded, importing this module raises, and every device entry point needs a
CUDA tensor. Build it with ``python -m paper_2307_07950_b200._build``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (
    POINTER,
    Structure,
    c_char_p,
    c_double,
    c_float,
    c_int,
    c_int32,
    c_int64,
    c_void_p,
)
from pathlib import Path

from .errors import ConfigError, SignalError

# SS_LIB_PATH: load another build of the library (A/B timing of two builds on one box)
LIB_PATH = Path(os.environ.get("SS_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libselsync_b200.so")

SS_OK, SS_ERR_CONFIG, SS_ERR_SIGNAL, SS_ERR_CUDA = 0, 1, 2, 3
SS_FLAG_SYNC, SS_FLAG_ERR_NAN, SS_FLAG_ERR_NEG = 1, 2, 4


class NativeError(RuntimeError):
    """CUDA launch/runtime failure reported by the library (SS_ERR_CUDA)."""


class SignalStateC(Structure):
    """ss_signal_state (64 bytes) -- GradSignalState, signal.py:41-61."""

    _fields_ = [
        ("smoothing", c_double),
        ("ewma_current", c_double),
        ("ewma_previous", c_double),
        ("max_delta_seen", c_double),
        ("last_delta", c_double),
        ("last_norm_sq", c_double),
        ("step_count", c_int64),
        ("warmup", c_int32),
        ("error", c_int32),
    ]


class TraceRowC(Structure):
    """ss_trace_row (32 bytes)."""

    _fields_ = [
        ("grad_norm_sq", c_double),
        ("ewma", c_double),
        ("delta_g", c_double),
        ("step", c_int32),
        ("word", c_int32),
    ]


SYMM_MAX_RANKS = 16
ORDER_EARLY_VOTE = 0x10  # SS_ORDER_EARLY_VOTE: order_mode flag, the exact early vote (opt-in)


class SymmGroupC(Structure):
    """ss_symm_group -- a rank's view of the symmetric buffer and signal slots."""

    _fields_ = [
        ("bufs", c_void_p * SYMM_MAX_RANKS),
        ("pads", c_void_p * SYMM_MAX_RANKS),
        ("mc", c_void_p),
        ("seq", c_void_p),
        ("agreed_ring", c_void_p),
        ("err", c_void_p),
        ("timeout_s", c_double),
        ("rank", c_int32),
        ("world", c_int32),
        ("ring_cap", c_int32),
        ("max_blocks", c_int32),
        ("order_mode", c_int32),
        ("order_threshold", c_float),
        ("tile_cnt", c_void_p * SYMM_MAX_RANKS),
        ("epoch", c_void_p),
        ("predictor", c_void_p),
        ("tile_elems", c_int64),
        ("n_tiles", c_int64),
        ("tile_norm", c_void_p),
        ("debug_events", c_void_p),
        ("debug_cap", c_int64),
    ]


class RankStepC(Structure):
    """ss_rank_step -- one rank's step arguments (pointers + hyperparameters): a
    colocated rank's, or the input of ss_step_plan_init."""

    _fields_ = [
        ("w", c_void_p), ("g", c_void_p), ("m", c_void_p), ("n", c_int64),
        ("momentum", c_float), ("dampening", c_float), ("weight_decay", c_float), ("nesterov", c_int32),
        ("st", c_void_p), ("delta", c_double), ("word", c_void_p), ("trace", c_void_p),
        ("trace_cap", c_int32), ("reserved", c_int32), ("group", c_void_p), ("ws", c_void_p),
    ]


class ColocatedPlanC(Structure):
    """ss_colocated_plan."""

    _fields_ = [("args_dev", c_void_p), ("ranks", c_int32), ("blocks_per_rank", c_int32), ("grads", c_int32),
                ("flags", c_int32)]


STEP_PLAN_WORDS = 192  # SS_STEP_PLAN_WORDS


class StepPlanC(Structure):
    """ss_step_plan -- opaque storage of a prepared per-rank step."""

    _fields_ = [("opaque", ctypes.c_uint64 * STEP_PLAN_WORDS)]


_P = c_void_p
_SIGS = {
    "ss_abi_version": ([], c_int),
    "ss_last_error": ([], c_char_p),
    "ss_signal_state_size": ([], c_int),
    "ss_trace_row_size": ([], c_int),
    "ss_default_smoothing": ([c_int32, POINTER(c_double)], c_int),
    "ss_check_delta": ([c_double], c_int),
    "ss_signal_init": ([POINTER(SignalStateC), c_double, c_int32], c_int),
    "ss_signal_observe": ([POINTER(SignalStateC), c_double], c_int),
    "ss_relative_change": ([POINTER(SignalStateC), POINTER(c_double)], c_int),
    "ss_decide": ([POINTER(SignalStateC), c_double, POINTER(c_int32)], c_int),
    "ss_sync_known_ahead": ([POINTER(SignalStateC), c_double, POINTER(c_int32)], c_int),
    "ss_sync_proven_early": ([POINTER(SignalStateC), c_double, c_double, POINTER(c_int32)], c_int),
    "ss_workspace_bytes": ([POINTER(c_int64)], c_int),
    "ss_workspace_reset": ([_P, _P], c_int),
    "ss_norm_sq_f32": ([_P, c_int64, _P, _P, _P], c_int),
    "ss_norm_sq_multi_f32": (
        [POINTER(c_void_p), POINTER(c_int64), c_int32, _P, _P, c_double, _P, _P, c_int32, _P, _P],
        c_int,
    ),
    "ss_signal_step": ([_P, _P, c_double, _P, _P, c_int32, _P], c_int),
    "ss_norm_signal_f32": ([_P, c_int64, _P, c_double, _P, _P, c_int32, _P, _P], c_int),
    "ss_sgd_update_f32": (
        [_P, _P, _P, c_int64, c_float, c_float, c_float, c_float, c_int32, c_int32, _P, c_float, _P],
        c_int,
    ),
    "ss_update_norm_signal_f32": (
        [_P, _P, _P, c_int64, c_float, c_float, c_float, c_float, c_int32, c_int32,
         _P, c_double, _P, _P, c_int32, _P, _P],
        c_int,
    ),
    "ss_sgd_update_multi_f32": (
        [POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_int64), c_int32, c_float, c_float,
         c_float, c_float, c_int32, c_int32, _P, c_float, _P],
        c_int,
    ),
    "ss_update_norm_signal_multi_f32": (
        [POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_int64), c_int32, c_float, c_float,
         c_float, c_float, c_int32, c_int32, _P, c_double, _P, _P, c_int32, _P, _P],
        c_int,
    ),
    "ss_replica_average_f32": ([POINTER(c_void_p), c_int32, c_int64, _P], c_int),
    "ss_replica_sum_f32": ([POINTER(c_void_p), c_int32, c_int64, _P], c_int),
    "ss_mean_f32": ([POINTER(c_void_p), c_int32, c_int64, _P, _P], c_int),
    "ss_replica_flag_max_i32": ([POINTER(c_void_p), c_int32, _P], c_int),
    "ss_symm_signal_bytes": ([c_int32, POINTER(c_int64)], c_int),
    "ss_symm_group_layout": ([POINTER(c_int64), c_int32, POINTER(c_int32)], c_int),
    "ss_symm_sync_f32": ([POINTER(SymmGroupC), c_int64, _P, c_int32, c_float, _P, _P], c_int),
    "ss_step_symm_ga_f32": (
        [_P, _P, _P, c_int64, c_float, c_float, c_float, c_float, c_int32, c_int32,
         _P, c_double, _P, _P, c_int32, POINTER(SymmGroupC), _P, _P],
        c_int,
    ),
    "ss_colocated_args_bytes": ([c_int32, POINTER(c_int64)], c_int),
    "ss_colocated_prepare_f32": ([c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p], c_int),
    "ss_colocated_step_f32": ([c_void_p, c_float, c_int32, c_void_p], c_int),
    "ss_rank_step_layout": ([POINTER(c_int64), c_int32, POINTER(c_int32)], c_int),
    "ss_step_plan_init": ([c_void_p, c_void_p, c_int32], c_int),
    "ss_step_plan_launch": ([c_void_p, c_void_p, c_float, c_int32, c_void_p], c_int),
    "ss_step_symm_f32": (
        [_P, _P, _P, c_int64, c_float, c_float, c_float, c_float, c_int32, c_int32,
         _P, c_double, _P, _P, c_int32, POINTER(SymmGroupC), _P, _P],
        c_int,
    ),
}

EXPORTED = tuple(_SIGS)


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the SelSync B200 path has no CPU fallback. "
            "Build it with `python -m paper_2307_07950_b200._build` (nvcc, sm_100a)."
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.ss_abi_version() != 1:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.ss_abi_version()} != 1")
    if lib.ss_signal_state_size() != ctypes.sizeof(SignalStateC):
        raise ImportError("ss_signal_state layout mismatch")
    if lib.ss_trace_row_size() != ctypes.sizeof(TraceRowC):
        raise ImportError("ss_trace_row layout mismatch")
    return lib


LIB = _load()


def check(rc: int) -> None:
    """Map a status code onto the reference's exception types (errors.py:4-17)."""
    if rc == SS_OK:
        return
    msg = (LIB.ss_last_error() or b"").decode(errors="replace")
    if rc == SS_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == SS_ERR_SIGNAL:
        raise SignalError(msg)
    raise NativeError(msg)


def workspace_bytes() -> int:
    out = c_int64(0)
    check(LIB.ss_workspace_bytes(ctypes.byref(out)))
    return int(out.value)


def ptr_array(ptrs) -> ctypes.Array:
    arr = (c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr

