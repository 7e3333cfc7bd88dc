"""Rank-group collectives of the SelSync step over torch.distributed.

The reference relays everything through a parameter server (runtime.py:
``_on_flags`` :319-333 for the flag OR, ``_close_round`` :275-294 for the
parameter mean). Here there is no server: one process per GPU, NCCL over
NVLink/NVSwitch, and two collectives per step --

  C1  ``agree``:    allreduce(int32[1], MAX) of the flag word, every step
  C2  ``average_``: allreduce(fp32[P], AVG) (or SUM after a 1/N pre-scale)

Collectives are issued on the caller's current CUDA stream ordering (torch's
ProcessGroupNCCL makes its NCCL stream wait on it and the current stream wait
on the result; no host synchronisation). The same class runs over ``gloo`` on
CPU tensors, which the world-size-2 CPU tests use.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch
import torch.distributed as dist

from .errors import ConfigError, TransportError


class RankGroup:
    def __init__(self, group: Optional[dist.ProcessGroup] = None):
        if not (dist.is_available() and dist.is_initialized()):
            self.group = None
            self.size = 1
            self.rank = 0
            self.backend = None
            return
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = str(dist.get_backend(group)).lower()

    @property
    def distributed(self) -> bool:
        return self.size > 1

    def _call(self, fn, *args, **kw):
        try:
            return fn(*args, group=self.group, **kw)
        except RuntimeError as exc:  # NCCL / gloo failures surface as RuntimeError
            raise TransportError(str(exc)) from exc

    def agree(self, word: torch.Tensor) -> None:
        """C1: every rank ends with the MAX of the words == OR of the votes."""
        if word.dtype != torch.int32 or word.numel() != 1:
            raise ConfigError("flag word must be a single int32")
        if self.distributed:
            self._call(dist.all_reduce, word, op=dist.ReduceOp.MAX)

    def average_(self, buf: torch.Tensor) -> None:
        """C2: in-place mean over ranks (aggregate_mean, strategies.py:159-168)."""
        if not self.distributed:
            return
        if self.backend == "nccl":
            self._call(dist.all_reduce, buf, op=dist.ReduceOp.AVG)
        else:  # gloo has no AVG
            self._call(dist.all_reduce, buf, op=dist.ReduceOp.SUM)
            buf.div_(self.size)

    def sum_(self, buf: torch.Tensor) -> None:
        """C2 after the 1/N pre-scale fused into the update epilogue."""
        if self.distributed:
            self._call(dist.all_reduce, buf, op=dist.ReduceOp.SUM)

    def broadcast_(self, buf: torch.Tensor, src_rank: int = 0) -> None:
        """Bootstrap: replicas start identical (runtime.py:178-191)."""
        if self.distributed:
            src = dist.get_global_rank(self.group, src_rank) if self.group is not None else src_rank
            self._call(dist.broadcast, buf, src=src)

    def max_float(self, value: float, device) -> float:
        """Max of a host scalar over ranks (bench timing: max over ranks)."""
        if not self.distributed:
            return float(value)
        t = torch.tensor([float(value)], dtype=torch.float64, device=device)
        self._call(dist.all_reduce, t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make_symmetric(self, numel: int, device, **kw) -> "SymmetricParams":
        """This rank's view of a symmetric parameter buffer (torch symmetric memory)."""
        return SymmetricParams(numel, device, self, **kw)

    def barrier(self, device=None) -> None:
        if self.distributed:
            if self.backend == "nccl" and device is not None:
                self._call(dist.barrier, device_ids=[torch.device(device).index])
            else:
                self._call(dist.barrier)


SIGNAL_OFFSET = 8192  # our slots sit at the top of torch's 9216-byte signal pad

ORDERS = {"update_first": 0, "norm_first": 1, "adaptive": 2, "nan_safe": 3}


def resolve_order(order: str, numel: int, world: int) -> str:
    """order="auto" (the default): "adaptive" where the ticketed norm-first
    pass pays on sync steps, else "update_first". Measured on B200 (bench
    modes, P sweep, profiles/r02_order_size/): at N = 2 update-first is faster
    up to 16M parameters and adaptive from 32M; at N = 4 update-first wins
    at 4M, adaptive from 16M (the mean costs more bytes per link there, so
    overlapping it pays earlier)."""
    if order != "auto":
        return order
    return "adaptive" if numel >= (24_000_000 if world <= 2 else 10_000_000) else "update_first"


def default_tile_elems(numel: int) -> int:
    # measured (N = 2, one graph replay per step): 4096-element tiles win
    # below ~2M parameters (more tiles than blocks), 16384 from 4M up
    return 4096 if numel <= (1 << 21) else 16384


class SymmetricView:
    """One rank's view of a symmetric (peer-addressable) flat fp32 buffer and
    of the per-rank device state the exchange kernels need, packed into the
    C struct ``ss_symm_group``. Subclasses provide the peer addresses: torch
    symmetric memory across GPUs (:class:`SymmetricParams`) or same-device
    buffers of ranks that share one GPU (``colocated.ColocatedSymmetric``)."""

    ORDERS = ORDERS

    def _fill_group(self, *, numel: int, rank: int, world: int, bufs, pads, mc, tile_cnt,
                    ring_capacity: int, timeout_s: float, order: str, order_threshold: float,
                    tile_elems: int, max_blocks: int = 0) -> None:
        from . import _native as N

        if world > N.SYMM_MAX_RANKS:
            raise ConfigError(f"at most {N.SYMM_MAX_RANKS} ranks per symmetric group")
        if order not in ORDERS:
            raise ConfigError(f"order must be one of {sorted(ORDERS)}, got {order!r}")
        if tile_elems <= 0 or tile_elems % 4:
            raise ConfigError("tile_elems must be a positive multiple of 4")
        if max_blocks < 0:
            raise ConfigError(f"max_blocks must be >= 0, got {max_blocks}")
        self.rank, self.world = int(rank), int(world)
        self.multicast = bool(mc)
        self.mc = mc or None
        self.seq = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.ring_capacity = int(ring_capacity)
        self.agreed = torch.zeros(self.ring_capacity, dtype=torch.int32, device=self.device)
        self.timeout_s = float(timeout_s)
        self.order = order
        self.n_tiles = (numel + tile_elems - 1) // tile_elems
        g = N.SymmGroupC()
        for r, p in enumerate(bufs):
            g.bufs[r] = int(p)
        for r, p in enumerate(pads):
            g.pads[r] = int(p)
        for r, p in enumerate(tile_cnt):
            g.tile_cnt[r] = int(p)
        g.mc = self.mc
        g.seq = self.seq.data_ptr()
        g.agreed_ring = self.agreed.data_ptr()
        g.err = self.err.data_ptr()
        g.timeout_s = self.timeout_s
        g.rank, g.world, g.ring_cap = self.rank, self.world, self.ring_capacity
        g.max_blocks = int(max_blocks)
        # order of the one-launch step; the norm-first order overlaps the update
        # with the mean on sync steps and needs per-tile arrival counters
        g.order_mode = ORDERS[order]
        g.order_threshold = float(order_threshold)
        # known-sync pass (warmup steps, delta == 0): ||g||^2 partial per update
        # tile; SS_KNOWN_SYNC=0 disables the pass (A/B knob)
        self.tile_norm = None
        if os.environ.get("SS_KNOWN_SYNC", "1") != "0":
            self.tile_norm = torch.zeros(max(1, self.n_tiles), dtype=torch.float64, device=self.device)
            g.tile_norm = self.tile_norm.data_ptr()
        self.epoch = torch.zeros(1, dtype=torch.int32, device=self.device)
        # order predictor: P(sync) per context of the last two agreed decisions + the context
        self.predictor = torch.zeros(5, dtype=torch.float32, device=self.device)
        g.epoch = self.epoch.data_ptr()
        g.predictor = self.predictor.data_ptr()
        g.tile_elems = int(tile_elems)
        g.n_tiles = int(self.n_tiles)
        self.group_c = g
        self.group_ref = ctypes.byref(g)
        self.version = 0  # bumped on every change of group_c (prepared step plans read it once)

    def set_early_vote(self, on: bool) -> None:
        """Exact early vote of the norm-first orders (opt-in): the
        mean starts once a running lower bound of ||g||^2 proves the vote sync."""
        from . import _native as N

        self.group_c.order_mode = ORDERS[self.order] | (N.ORDER_EARLY_VOTE if on else 0)
        self.version += 1

    def sync_(self, word: torch.Tensor, ws_ptr: int, *, exchange: bool, stream: int) -> None:
        from . import _native as N

        N.check(N.LIB.ss_symm_sync_f32(self.group_ref, self.buf.numel(), word.data_ptr(), int(exchange),
                                       1.0 / self.world, ws_ptr, stream))

    def enable_timeline(self, capacity: int) -> torch.Tensor:
        """Record the per-ticket timeline of the overlapped sync step (tooling):
        4 x int64 per ticket {kind << 48 | tile, t_start, t_ready, t_end} (ns)."""
        # + 8 markers: step start, vote posted, votes in, -, last arrival, barrier done
        self.timeline = torch.zeros(4 * int(capacity) + 8, dtype=torch.int64, device=self.device)
        self.group_c.debug_events = self.timeline.data_ptr()
        self.group_c.debug_cap = int(capacity)
        self.version += 1
        return self.timeline

    @property
    def one_launch_capable(self) -> bool:
        """The fused one-launch step supports NVLS or P2P widths 1, 2, 4, 8."""
        return self.multicast or self.world in (1, 2, 4, 8)

    def check(self) -> None:
        if int(self.err.item()) != 0:
            raise TransportError("a peer did not answer the device-side exchange within "
                                 f"{self.timeout_s:.0f} s")


class SymmetricParams(SymmetricView):
    """Flat fp32 buffer in symmetric (peer-mapped) memory + the device-side
    SelSync exchange kernels over it.

    Allocation and address exchange use torch.distributed._symmetric_memory
    (plumbing); the data path is our kernels: optional P2P flag exchange, then
    -- only when the agreed flag word says sync -- the parameter mean written
    into every rank's buffer (NVLS multimem when the switch supports it, P2P
    loads/stores otherwise), with no host involvement.
    """

    def __init__(self, numel: int, device, comm: RankGroup, *, ring_capacity: int = 1 << 14,
                 timeout_s: float = 30.0, use_multicast="auto", order: str = "update_first",
                 order_threshold: float = 0.2, tile_elems: Optional[int] = None, max_blocks: int = 0):
        import torch.distributed._symmetric_memory as symm_mem

        from . import _native as N

        if not dist.is_initialized():
            raise ConfigError("symmetric memory needs an initialised process group")
        self.device = torch.device(device)
        self.comm = comm
        group = comm.group if comm.group is not None else dist.group.WORLD
        self.buf = symm_mem.empty(numel, dtype=torch.float32, device=self.device)
        self.hdl = symm_mem.rendezvous(self.buf, group)
        world = int(self.hdl.world_size)
        rank = int(self.hdl.rank)
        need = ctypes.c_int64(0)
        N.check(N.LIB.ss_symm_signal_bytes(world, ctypes.byref(need)))
        if SIGNAL_OFFSET + need.value > int(self.hdl.signal_pad_size):
            raise ConfigError("signal pad too small for the exchange slots")
        # NVLS moves 4P(1 + 1/N) bytes per link direction, the P2P two-shot
        # 2(N-1)/N * 4P: multicast wins from N = 4 up (measured on B200:
        # N=2 P2P 603 us vs NVLS 1030 us; N=4 NVLS 897 us vs P2P 920 us at 400 MB)
        if use_multicast == "auto":
            use_multicast = world >= 4
        mc = int(self.hdl.multicast_ptr) if use_multicast else 0
        # our slots of the local pad start zeroed; everyone zeroes before anyone posts
        pad = self.hdl.get_signal_pad(rank, [need.value // 8], torch.int64, SIGNAL_OFFSET // 8)
        pad.zero_()
        if tile_elems is None:
            tile_elems = default_tile_elems(numel)
        n_tiles = (numel + max(int(tile_elems), 1) - 1) // max(int(tile_elems), 1)
        self.cnt = symm_mem.empty(max(1, n_tiles), dtype=torch.int32, device=self.device)
        self.cnt_hdl = symm_mem.rendezvous(self.cnt, group)
        self.cnt.zero_()
        self._fill_group(numel=numel, rank=rank, world=world, bufs=self.hdl.buffer_ptrs,
                         pads=[int(p) + SIGNAL_OFFSET for p in self.hdl.signal_pad_ptrs], mc=mc,
                         tile_cnt=self.cnt_hdl.buffer_ptrs, ring_capacity=ring_capacity,
                         timeout_s=timeout_s, order=order, order_threshold=order_threshold,
                         tile_elems=int(tile_elems), max_blocks=max_blocks)
        torch.cuda.synchronize(self.device)
        comm.barrier(self.device)
