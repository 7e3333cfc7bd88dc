"""Tensor-level wrappers of the sm_100a kernels (C-ABI: include/selsync_b200.h).

Every function validates its tensors (CUDA, dtype, contiguity, sizes) and then
launches on the device's *current* torch stream. There is no CPU path: a CPU
tensor raises ConfigError. ``LAUNCHES`` counts kernel launches issued through
this module (bench.py reports it as ``gpu_launches``).
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, SignalError

LAUNCHES = 0

TRACE_DTYPE = np.dtype(
    [("grad_norm_sq", "<f8"), ("ewma", "<f8"), ("delta_g", "<f8"), ("step", "<i4"), ("word", "<i4")]
)
STATE_DTYPE = np.dtype(
    [
        ("smoothing", "<f8"),
        ("ewma_current", "<f8"),
        ("ewma_previous", "<f8"),
        ("max_delta_seen", "<f8"),
        ("last_delta", "<f8"),
        ("last_norm_sq", "<f8"),
        ("step_count", "<i8"),
        ("warmup", "<i4"),
        ("error", "<i4"),
    ]
)
assert TRACE_DTYPE.itemsize == ctypes.sizeof(N.TraceRowC) == 32
assert STATE_DTYPE.itemsize == ctypes.sizeof(N.SignalStateC) == 64


def _count(k: int = 1) -> None:
    global LAUNCHES
    LAUNCHES += k


def stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _need(t: Optional[torch.Tensor], dtype, name: str, device=None) -> None:
    if t is None:
        raise ConfigError(f"{name} is required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ConfigError(f"{name} must be a CUDA tensor (the B200 path has no CPU fallback)")
    if t.dtype != dtype:
        raise ConfigError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ConfigError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ConfigError(f"{name} is on {t.device}, expected {device}")


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Workspace:
    """Block-partial scratch + arrival counter for the reduction kernels.

    One workspace per stream; it is zeroed once and self-resets at the end of
    every reduction launch (also across CUDA-graph replays)."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.buf = torch.zeros(N.workspace_bytes(), dtype=torch.uint8, device=self.device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()


class DeviceSignal:
    """Device-resident GradSignalState + flag word + decision-trace ring."""

    def __init__(self, device, smoothing: float, warmup: int, trace_capacity: int = 4096):
        if trace_capacity < 1:
            raise ConfigError("trace_capacity must be >= 1")
        self.device = torch.device(device)
        c = N.SignalStateC()
        N.check(N.LIB.ss_signal_init(ctypes.byref(c), float(smoothing), int(warmup)))
        host = torch.frombuffer(bytearray(bytes(c)), dtype=torch.uint8)
        self.state = host.to(self.device)
        self.word = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.trace_capacity = int(trace_capacity)
        self.trace = torch.zeros(self.trace_capacity * TRACE_DTYPE.itemsize, dtype=torch.uint8,
                                 device=self.device)

    def read_state(self) -> np.void:
        return np.frombuffer(self.state.cpu().numpy().tobytes(), dtype=STATE_DTYPE)[0]

    def read_trace(self) -> np.ndarray:
        return np.frombuffer(self.trace.cpu().numpy().tobytes(), dtype=TRACE_DTYPE).copy()


# ---------------------------------------------------------------- K1


def norm_sq(g: torch.Tensor, out: Optional[torch.Tensor] = None,
            ws: Optional[Workspace] = None) -> torch.Tensor:
    """||g||^2 (fp64, device) of a flat fp32 tensor -- float(grad @ grad), strategies.py:285."""
    _need(g, torch.float32, "g")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=g.device)
    _need(out, torch.float64, "out", g.device)
    ws = ws or Workspace(g.device)
    N.check(N.LIB.ss_norm_sq_f32(g.data_ptr(), g.numel(), out.data_ptr(), ws.ptr, stream_of(g)))
    _count()
    return out


def norm_sq_multi(tensors: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None,
                  ws: Optional[Workspace] = None, signal: Optional[DeviceSignal] = None,
                  delta: float = 0.0) -> torch.Tensor:
    """||g||^2 over a list of fp32 tensors (the model's separate p.grad tensors)."""
    if not tensors:
        raise ConfigError("norm_sq_multi needs at least one tensor")
    dev = tensors[0].device
    for i, t in enumerate(tensors):
        _need(t, torch.float32, f"tensors[{i}]", dev)
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=dev)
    ws = ws or Workspace(dev)
    ptrs = N.ptr_array([t.data_ptr() for t in tensors])
    sizes = (ctypes.c_int64 * len(tensors))(*[t.numel() for t in tensors])
    st = signal.state.data_ptr() if signal else None
    word = signal.word.data_ptr() if signal else None
    trace = signal.trace.data_ptr() if signal else None
    cap = signal.trace_capacity if signal else 0
    N.check(N.LIB.ss_norm_sq_multi_f32(ptrs, sizes, len(tensors), out.data_ptr(), st, float(delta),
                                       word, trace, cap, ws.ptr, stream_of(tensors[0])))
    _count((len(tensors) + 255) // 256)
    return out


# ---------------------------------------------------------------- K2


def signal_step(signal: DeviceSignal, norm_sq_dev: torch.Tensor, delta: float) -> None:
    _need(norm_sq_dev, torch.float64, "norm_sq", signal.device)
    N.check(N.LIB.ss_signal_step(signal.state.data_ptr(), norm_sq_dev.data_ptr(), float(delta),
                                 signal.word.data_ptr(), signal.trace.data_ptr(),
                                 signal.trace_capacity, stream_of(norm_sq_dev)))
    _count()


def norm_signal(g: torch.Tensor, signal: DeviceSignal, delta: float, ws: Workspace) -> None:
    """K1 + K2 in one launch."""
    _need(g, torch.float32, "g", signal.device)
    N.check(N.LIB.ss_norm_signal_f32(g.data_ptr(), g.numel(), signal.state.data_ptr(), float(delta),
                                     signal.word.data_ptr(), signal.trace.data_ptr(),
                                     signal.trace_capacity, ws.ptr, stream_of(g)))
    _count()


# ---------------------------------------------------------------- K3 / K13


def _sgd_check(w, g, m, momentum):
    _need(w, torch.float32, "w")
    _need(g, torch.float32, "g", w.device)
    if g.numel() != w.numel():
        raise ConfigError("gradient shape does not match parameter vector")
    if momentum != 0.0:
        _need(m, torch.float32, "momentum buffer", w.device)
        if m.numel() != w.numel():
            raise ConfigError("momentum buffer size does not match parameter vector")


def sgd_update_(w, g, m=None, *, lr: float, momentum: float = 0.0, dampening: float = 0.0,
                weight_decay: float = 0.0, nesterov: bool = False, first_step: bool = False,
                sync_word: Optional[torch.Tensor] = None, sync_scale: float = 1.0) -> None:
    """K3 in place (model.py:215-221 with the torch.optim.SGD extension)."""
    _sgd_check(w, g, m, momentum)
    if sync_word is not None:
        _need(sync_word, torch.int32, "sync_word", w.device)
    N.check(N.LIB.ss_sgd_update_f32(
        w.data_ptr(), g.data_ptr(), _ptr(m) if momentum != 0.0 else None, w.numel(), float(lr),
        float(momentum), float(dampening), float(weight_decay), int(bool(nesterov)),
        int(bool(first_step)), _ptr(sync_word), float(sync_scale), stream_of(w)))
    _count()


def update_norm_signal_(w, g, m, signal: DeviceSignal, ws: Workspace, *, lr: float, delta: float,
                        momentum: float = 0.0, dampening: float = 0.0, weight_decay: float = 0.0,
                        nesterov: bool = False, first_step: bool = False) -> None:
    """K13 + K2: one pass over (w, g, m) that also produces ||g||^2 and the vote."""
    _sgd_check(w, g, m, momentum)
    N.check(N.LIB.ss_update_norm_signal_f32(
        w.data_ptr(), g.data_ptr(), _ptr(m) if momentum != 0.0 else None, w.numel(), float(lr),
        float(momentum), float(dampening), float(weight_decay), int(bool(nesterov)),
        int(bool(first_step)), signal.state.data_ptr(), float(delta), signal.word.data_ptr(),
        signal.trace.data_ptr(), signal.trace_capacity, ws.ptr, stream_of(w)))
    _count()


# ---------------------------------------------------------------- replicas


def replica_average_(bufs: Sequence[torch.Tensor], divide: bool = True) -> None:
    """aggregate_mean over replica buffers, written back into every replica
    (divide=False: the plain sum, for buffers pre-scaled by 1/N)."""
    if not bufs:
        raise ConfigError("need at least one replica")
    dev = bufs[0].device
    n = bufs[0].numel()
    for i, b in enumerate(bufs):
        _need(b, torch.float32, f"replica[{i}]", dev)
        if b.numel() != n:
            raise ConfigError("aggregate_mean: layout mismatch")
    fn = N.LIB.ss_replica_average_f32 if divide else N.LIB.ss_replica_sum_f32
    N.check(fn(N.ptr_array([b.data_ptr() for b in bufs]), len(bufs), n, stream_of(bufs[0])))
    _count()


def mean(bufs: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None) -> torch.Tensor:
    if not bufs:
        raise ConfigError("aggregate_mean needs at least one vector")
    dev = bufs[0].device
    n = bufs[0].numel()
    for i, b in enumerate(bufs):
        _need(b, torch.float32, f"vectors[{i}]", dev)
        if b.numel() != n:
            raise ConfigError("aggregate_mean: layout mismatch")
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=dev)
    _need(out, torch.float32, "out", dev)
    N.check(N.LIB.ss_mean_f32(N.ptr_array([b.data_ptr() for b in bufs]), len(bufs), n,
                              out.data_ptr(), stream_of(out)))
    _count()
    return out


def replica_flag_max_(words: Sequence[torch.Tensor]) -> None:
    dev = words[0].device
    for i, w in enumerate(words):
        _need(w, torch.int32, f"word[{i}]", dev)
    N.check(N.LIB.ss_replica_flag_max_i32(N.ptr_array([w.data_ptr() for w in words]), len(words),
                                          stream_of(words[0])))
    _count()


def raise_for_word(word: int, where: str = "") -> None:
    """Turn the error bits of an agreed flag word (>= 2) into the reference's
    SignalError (signal.py:67-70); a NaN anywhere wins over a negative."""
    if word & N.SS_FLAG_ERR_NEG and not word & N.SS_FLAG_ERR_NAN:
        raise SignalError(f"squared norm cannot be negative{where}")
    raise SignalError(f"observed a NaN gradient norm{where}")


def step_symm_(w, g, m, signal: DeviceSignal, ws: Workspace, group, *, lr: float, delta: float,
               momentum: float = 0.0, dampening: float = 0.0, weight_decay: float = 0.0,
               nesterov: bool = False, first_step: bool = False) -> None:
    """The whole SelSync step in one cooperative launch (``ss_step_symm_f32``):
    update + ||g||^2 + signal + P2P vote exchange + conditional NVLink mean.
    ``group`` is a :class:`collectives.SymmetricParams`; ``w`` its buffer."""
    _sgd_check(w, g, m, momentum)
    if w.data_ptr() != group.buf.data_ptr():
        raise ConfigError("w must be the symmetric parameter buffer")
    N.check(N.LIB.ss_step_symm_f32(
        w.data_ptr(), g.data_ptr(), _ptr(m) if momentum != 0.0 else None, w.numel(), float(lr),
        float(momentum), float(dampening), float(weight_decay), int(bool(nesterov)),
        int(bool(first_step)), signal.state.data_ptr(), float(delta), signal.word.data_ptr(),
        signal.trace.data_ptr(), signal.trace_capacity, group.group_ref, ws.ptr, stream_of(w)))
    _count()


def _tensor_table(ws, gs, ms, momentum):
    if not ws or len(ws) != len(gs) or (momentum != 0.0 and (ms is None or len(ms) != len(ws))):
        raise ConfigError("parameter / gradient / momentum lists must have equal lengths")
    dev = ws[0].device
    for i, (w, g) in enumerate(zip(ws, gs)):
        _need(w, torch.float32, f"params[{i}]", dev)
        _need(g, torch.float32, f"grads[{i}]", dev)
        if g.numel() != w.numel():
            raise ConfigError(f"gradient {i} does not match its parameter")
        if momentum != 0.0:
            _need(ms[i], torch.float32, f"momentum[{i}]", dev)
            if ms[i].numel() != w.numel():
                raise ConfigError(f"momentum buffer {i} does not match its parameter")
    wp = N.ptr_array([w.data_ptr() for w in ws])
    gp = N.ptr_array([g.data_ptr() for g in gs])
    mp = N.ptr_array([m.data_ptr() for m in ms]) if momentum != 0.0 else N.ptr_array([0] * len(ws))
    sizes = (ctypes.c_int64 * len(ws))(*[w.numel() for w in ws])
    return wp, gp, mp, sizes


def sgd_update_multi_(ws, gs, ms=None, *, lr: float, momentum: float = 0.0, dampening: float = 0.0,
                      weight_decay: float = 0.0, nesterov: bool = False, first_step: bool = False,
                      sync_word: Optional[torch.Tensor] = None, sync_scale: float = 1.0) -> None:
    """K3 over a tensor list (pointer table)."""
    wp, gp, mp, sizes = _tensor_table(ws, gs, ms, momentum)
    N.check(N.LIB.ss_sgd_update_multi_f32(
        wp, gp, mp, sizes, len(ws), float(lr), float(momentum), float(dampening), float(weight_decay),
        int(bool(nesterov)), int(bool(first_step)), _ptr(sync_word), float(sync_scale), stream_of(ws[0])))
    _count((len(ws) + 127) // 128)


def update_norm_signal_multi_(ws, gs, ms, signal: DeviceSignal, workspace: Workspace, *, lr: float,
                              delta: float, momentum: float = 0.0, dampening: float = 0.0,
                              weight_decay: float = 0.0, nesterov: bool = False, first_step: bool = False) -> None:
    """K13 + K2 over a tensor list: one pass, ||g||^2 over all tensors, the vote."""
    wp, gp, mp, sizes = _tensor_table(ws, gs, ms, momentum)
    N.check(N.LIB.ss_update_norm_signal_multi_f32(
        wp, gp, mp, sizes, len(ws), float(lr), float(momentum), float(dampening), float(weight_decay),
        int(bool(nesterov)), int(bool(first_step)), signal.state.data_ptr(), float(delta),
        signal.word.data_ptr(), signal.trace.data_ptr(), signal.trace_capacity, workspace.ptr,
        stream_of(ws[0])))
    _count((len(ws) + 127) // 128)
