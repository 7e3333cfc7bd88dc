"""SelSync ranks that share ONE device: the multi-rank step kernels on one GPU.

Across GPUs each rank's parameters live in torch symmetric memory and the
one-launch step (``ss_step_symm_f32`` / ``ss_step_symm_ga_f32``) reads and
writes its peers' buffers over NVLink. Here the N ranks are N
``SelSyncStep`` objects on one device: every rank owns its own flat buffers,
signal slots, tile counters, step counter, predictor, agreed ring and
workspace, and its "peers" are the other ranks' same-device allocations --
exactly the ``ss_symm_group`` layout the kernels expect, with plain device
addresses instead of peer mappings.

Ranks whose kernels wait on one another must not be separate launches on one
GPU (nothing guarantees that they run at the same time), so the N ranks step
together in ONE cooperative launch (``ss_colocated_step_f32``): blocks
[r*G, (r+1)*G) run rank r's one-launch step over rank r's arguments -- the
same device code, per rank, as the per-GPU launch -- and the vote exchange,
the tile tickets, the mean and the end barrier run between the slices as they
do between GPUs (seq-tagged votes, release/acquire counters).

This is the reference's N-worker exchange (flag relay runtime.py:319-333,
mean round runtime.py:275-294 -> strategies.py:159-168, bootstrap
runtime.py:178-191) through the kernels a multi-GPU run uses, which a
single-GPU box can run and check against the reference's golden traces.
(The NVLS multicast path needs a multicast object over several GPUs and is
not reachable this way.)
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _native as N
from .collectives import SymmetricView, default_tile_elems
from .config import SelSyncConfig
from .errors import ConfigError


class ColocatedWorld:
    """Shared allocations of ``world`` ranks on one device: the N parameter
    (or gradient) buffers, the N signal regions and the N tile-counter arrays
    every rank's ``ss_symm_group`` points into."""

    def __init__(self, world: int, device):
        if world < 1 or world > N.SYMM_MAX_RANKS:
            raise ConfigError(f"world must be in [1, {N.SYMM_MAX_RANKS}], got {world}")
        self.world = int(world)
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ConfigError("colocated ranks need a CUDA device (no CPU fallback)")
        self.numel: Optional[int] = None
        self.views: dict[int, "ColocatedSymmetric"] = {}
        self.bcast: dict = {}

    def _allocate(self, numel: int, tile_elems: int) -> None:
        if self.numel is not None:
            if (numel, tile_elems) != (self.numel, self.tile_elems):
                raise ConfigError(f"every colocated rank needs the same buffer and tile size: "
                                  f"{(numel, tile_elems)} vs {(self.numel, self.tile_elems)}")
            return
        need = ctypes.c_int64(0)
        N.check(N.LIB.ss_symm_signal_bytes(self.world, ctypes.byref(need)))
        self.numel, self.tile_elems = int(numel), int(tile_elems)
        n_tiles = max(1, (numel + tile_elems - 1) // tile_elems)
        self.bufs = [torch.empty(numel, dtype=torch.float32, device=self.device) for _ in range(self.world)]
        self.pads = torch.zeros(self.world, need.value // 8, dtype=torch.int64, device=self.device)
        self.cnt = torch.zeros(self.world, n_tiles, dtype=torch.int32, device=self.device)

    def group(self, rank: int) -> "ColocatedGroup":
        if not 0 <= rank < self.world:
            raise ConfigError(f"rank {rank} out of range for {self.world} colocated ranks")
        return ColocatedGroup(self, rank)


class ColocatedGroup:
    """The ``RankGroup`` of one colocated rank. Votes and means travel inside
    the one-launch step kernels; there is no NCCL communicator, so only the
    symmetric-memory back end with the fused exchange is available."""

    backend = "colocated"

    def __init__(self, world: ColocatedWorld, rank: int):
        self.world_obj = world
        self.group = None
        self.size = world.world
        self.rank = int(rank)

    @property
    def distributed(self) -> bool:
        return self.size > 1

    def _no_host_collective(self, what: str):
        raise ConfigError(f"colocated ranks have no host collective ({what}); use collective='symm' "
                          "with flag_exchange='fused'")

    def agree(self, word: torch.Tensor) -> None:
        self._no_host_collective("flag allreduce")

    def average_(self, buf: torch.Tensor) -> None:
        self._no_host_collective("allreduce")

    def sum_(self, buf: torch.Tensor) -> None:
        self._no_host_collective("allreduce")

    def broadcast_(self, buf: torch.Tensor, src_rank: int = 0) -> None:
        """Bootstrap (runtime.py:178-191): every rank calls it with its own
        tensor of the same role (ranks are constructed in order); the source
        rank's call registers its tensor, the others copy it."""
        key = (src_rank, buf.numel(), buf.dtype)
        if self.rank == src_rank:
            self.world_obj.bcast[key] = buf
            return
        src = self.world_obj.bcast.get(key)
        if src is None:
            raise ConfigError(f"rank {src_rank} must broadcast before rank {self.rank} receives")
        buf.copy_(src)

    def max_float(self, value: float, device) -> float:
        return float(value)

    def barrier(self, device=None) -> None:
        pass

    def make_symmetric(self, numel: int, device, **kw) -> "ColocatedSymmetric":
        return ColocatedSymmetric(self.world_obj, self.rank, numel, device, **kw)


class ColocatedSymmetric(SymmetricView):
    """Rank ``rank``'s ``ss_symm_group`` over the shared same-device buffers."""

    def __init__(self, world: ColocatedWorld, rank: int, numel: int, device, *, ring_capacity: int = 1 << 14,
                 timeout_s: float = 10.0, use_multicast=False, order: str = "update_first",
                 order_threshold: float = 0.2, tile_elems: Optional[int] = None, max_blocks: int = 0):
        if use_multicast is True:
            raise ConfigError("colocated ranks have no multicast object (NVLS needs several GPUs)")
        self.device = torch.device(device)
        if self.device != world.device:
            raise ConfigError(f"rank on {self.device}, colocated world on {world.device}")
        if rank in world.views:
            raise ConfigError(f"colocated rank {rank} already has a symmetric buffer")
        if tile_elems is None:
            tile_elems = default_tile_elems(numel)
        world._allocate(int(numel), int(tile_elems))
        self.buf = world.bufs[rank]
        self._fill_group(numel=numel, rank=rank, world=world.world, bufs=[b.data_ptr() for b in world.bufs],
                         pads=[world.pads[r].data_ptr() for r in range(world.world)], mc=0,
                         tile_cnt=[world.cnt[r].data_ptr() for r in range(world.world)],
                         ring_capacity=ring_capacity, timeout_s=timeout_s, order=order,
                         order_threshold=order_threshold, tile_elems=int(tile_elems),
                         max_blocks=max_blocks)
        world.views[rank] = self


class ColocatedSelSync:
    """N SelSync ranks on one GPU, each a :class:`SelSyncStep` (state, trace,
    buffers), stepped together by ONE cooperative launch per step.

    API as :class:`ReplicaSelSync` (``set_grads`` / ``step`` / ``decisions`` /
    ``trace`` / ``params``): ``step(lr)`` enqueues the launch and returns;
    ``synchronize()`` waits and raises ``SignalError`` / ``TransportError`` as
    ``SelSyncStep`` does; ``capture(lr)`` records the launch as a CUDA graph.
    """

    def __init__(self, init_params: torch.Tensor, n_ranks: int, config: SelSyncConfig, *,
                 order: str = "adaptive", order_threshold: float = 0.2, tile_elems: Optional[int] = None,
                 timeout_s: float = 10.0, max_blocks: int = 0, trace_capacity: int = 4096,
                 nan_safe: bool = False, early_vote: bool = False):
        from .step import SelSyncStep

        if not isinstance(init_params, torch.Tensor) or not init_params.is_cuda:
            raise ConfigError("init_params must be a CUDA tensor")
        if n_ranks not in (1, 2, 4, 8):
            raise ConfigError(f"colocated ranks use the P2P widths 1, 2, 4, 8 of the step kernel, got {n_ranks}")
        p0 = init_params.reshape(-1).to(torch.float32)
        self.n = int(n_ranks)
        self.device = p0.device
        self.config = config
        self.world = ColocatedWorld(self.n, self.device)
        self.ranks: list = []
        for r in range(self.n):
            # only rank 0 holds the init; the others start from garbage and must
            # be overwritten by the bootstrap broadcast (runtime.py:178-191)
            init = p0.clone() if r == 0 else torch.full_like(p0, 7.0)
            st = SelSyncStep(init, torch.zeros_like(p0), config, group=self.world.group(r), collective="symm",
                             flag_exchange="fused", order=order, order_threshold=order_threshold,
                             tile_elems=tile_elems, timeout_s=timeout_s, trace_capacity=trace_capacity,
                             nan_safe=nan_safe, early_vote=early_vote)
            self.ranks.append(st)
        grads = config.aggregation == "grads"
        table = (N.RankStepC * self.n)()
        for r, st in enumerate(self.ranks):
            c = st.config
            table[r] = N.RankStepC(
                st.params.data_ptr(), st.grads.data_ptr(),
                st.momentum.data_ptr() if st.momentum is not None else None, st.params.numel(),
                float(c.momentum), float(c.dampening), float(c.weight_decay), int(bool(c.nesterov)),
                st.signal.state.data_ptr(), float(c.delta), st.signal.word.data_ptr(), st.signal.trace.data_ptr(),
                st.signal.trace_capacity, 0, ctypes.addressof(st.symm.group_c), st.ws.ptr)
        nbytes = ctypes.c_int64(0)
        N.check(N.LIB.ss_colocated_args_bytes(self.n, ctypes.byref(nbytes)))
        self._args = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
        self.plan = N.ColocatedPlanC(self._args.data_ptr(), 0, 0, 0, 0)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        N.check(N.LIB.ss_colocated_prepare_f32(ctypes.addressof(table), self.n, int(grads), int(max_blocks),
                                               ctypes.addressof(self.plan), stream))
        self.blocks_per_rank = int(self.plan.blocks_per_rank)
        torch.cuda.synchronize(self.device)

    @property
    def params(self) -> list:
        return [st.params for st in self.ranks]

    @property
    def grads(self) -> list:
        return [st.grads for st in self.ranks]

    def set_grads(self, grads: Sequence[torch.Tensor]) -> None:
        for st, g in zip(self.ranks, grads):
            st.grads.copy_(g.reshape(-1), non_blocking=True)

    def _launch(self, lr: float, stream) -> None:
        from . import kernels as K

        N.check(N.LIB.ss_colocated_step_f32(ctypes.addressof(self.plan), lr, int(self.steps_done == 0),
                                            stream.cuda_stream))
        K._count()

    def step(self, lr: float) -> None:
        """Enqueue one step of every rank (one launch, no host round-trip)."""
        lr = self.ranks[0]._check_lr(lr)
        self._launch(lr, torch.cuda.current_stream(self.device))
        for st in self.ranks:
            st._log_step(lr)

    def capture(self, lr: float) -> "CapturedColocatedStep":
        """Record one step of all ranks (the launch, this lr) as a CUDA graph."""
        if self.steps_done == 0:
            raise ConfigError("run one eager step first (the first step initialises the momentum buffers)")
        lr = self.ranks[0]._check_lr(lr)
        torch.cuda.synchronize(self.device)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self._launch(lr, torch.cuda.current_stream(self.device))
        torch.cuda.synchronize(self.device)
        return CapturedColocatedStep(self, graph, lr)

    def synchronize(self) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        for st in self.ranks:
            st.synchronize()

    @property
    def steps_done(self) -> int:
        return self.ranks[0].steps_done

    def decisions(self, rank: int = 0) -> list:
        return self.ranks[rank].decisions()

    def trace(self, rank: int):
        return self.ranks[rank].signal.read_trace()

    def records(self) -> list:
        return [row for st in self.ranks for row in st.records()]


class CapturedColocatedStep:
    def __init__(self, col: ColocatedSelSync, graph, lr: float):
        self.col, self.graph, self.lr = col, graph, lr

    def replay(self) -> None:
        from . import kernels as K

        self.graph.replay()
        for st in self.col.ranks:
            st._log_step(self.lr)
        K._count()
