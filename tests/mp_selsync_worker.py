"""torchrun worker for tests/test_multigpu.py: one rank per GPU, NCCL.

Runs SelSyncStep on a golden case (its N must equal WORLD_SIZE) and saves the
rank's decisions, trace rows and final parameters for the test to compare
with the reference's golden trace."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import _load_cases  # noqa: E402
from oracle import selsync_oracle as O  # noqa: E402
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402


def main():
    name, mode, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
    opts = {"fused": dict(collective="nccl", fuse=True),
            "prescale": dict(collective="nccl", fuse=False),
            "symm-nccl": dict(collective="symm", flag_exchange="nccl"),
            "symm-p2p": dict(collective="symm", flag_exchange="p2p"),
            "symm-fused": dict(collective="symm", flag_exchange="fused"),
            "symm-normfirst": dict(collective="symm", flag_exchange="fused", order="norm_first"),
            "symm-adaptive": dict(collective="symm", flag_exchange="fused", order="adaptive"),
            "symm-nansafe": dict(collective="symm", flag_exchange="fused", order="nan_safe")}[mode]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    c = _load_cases()[name]
    assert c["n"] == world, (c["n"], world)
    P = c["P"]
    # rank 0 holds the init; everyone else starts from garbage and must be
    # overwritten by the bootstrap broadcast (runtime.py:178-191)
    init = torch.tensor(c["init"], dtype=torch.float32, device=dev) if rank == 0 else \
        torch.full((P,), 7.0, device=dev)
    g = torch.zeros(P, device=dev)
    cfg = SelSyncConfig(delta=c["delta"], aggregation=c["aggregation"], warmup=c["warmup"],
                        smoothing=c["smoothing"])
    if c["aggregation"] != "params" and opts["collective"] == "symm" and opts.get("flag_exchange") != "fused":
        opts = dict(collective="nccl", fuse=True)
    step = SelSyncStep(init, g, cfg, **opts)
    host = [torch.from_numpy(O.synthetic_grad32(c["grad_seed"], rank, s, P)).pin_memory()
            for s in range(c["steps"])]
    g = step.grads  # gradient aggregation over symmetric memory owns the gradient buffer
    for s in range(c["steps"]):
        g.copy_(host[s], non_blocking=True)
        if step.async_capable and s % 2:
            step.step_async(c["lr"])  # device-side branch, no host round-trip
        else:
            step.step(c["lr"])
    step.synchronize()
    recs = step.records()
    np.savez(out / f"{name}_{mode}_rank{rank}.npz",
             decisions=np.array(step.decisions()), ewma=np.array([r["ewma"] for r in recs]),
             delta_g=np.array([np.nan if r["delta_g"] is None else r["delta_g"] for r in recs]),
             params=step.params.double().cpu().numpy(),
             multicast=np.array(bool(step.symm and step.symm.multicast)))
    dist.barrier()
    dist.destroy_process_group()


LARGE = dict(P=1_000_003, steps=14, seed=11, delta=0.05, warmup=2, smoothing=0.5, lr=0.05, momentum=0.9,
             weight_decay=4e-4, tile=4096)  # decisions: 8 sync, 4 local, 2 sync (>= 4.7% from a tie)


def large_init(seed, P):
    """w0 ~ U(-0.05, 0.05) in fp32; rank 0's copy is broadcast."""
    return np.random.default_rng(seed).uniform(-0.05, 0.05, P).astype(np.float32)


def large_aggregation(variant):
    return "grads" if variant.startswith("ga") else "params"


def large_delta(variant):
    """bsp: delta = 0, every step sync -- known before ||g||^2 (the known-sync pass)."""
    return 0.0 if variant == "bsp" else LARGE["delta"]


def large_main():
    """Many tiles and a ragged tail: P = 1,000,003 with 4096-element tiles
    (245 tiles, lag groups, a 3-element scalar tail), momentum + weight decay,
    mixed decisions; every step order / back end must give the oracle's trace."""
    variant, out = sys.argv[2], Path(sys.argv[3])
    opts = {"nccl": dict(collective="nccl", fuse=True),
            "update_first": dict(collective="symm", flag_exchange="fused", order="update_first"),
            "norm_first": dict(collective="symm", flag_exchange="fused", order="norm_first"),
            "adaptive": dict(collective="symm", flag_exchange="fused", order="adaptive"),
            "p2p-mean": dict(collective="symm", flag_exchange="fused", order="norm_first", multicast=False),
            "nvls-mean": dict(collective="symm", flag_exchange="fused", order="adaptive", multicast=True),
            "two-launch": dict(collective="symm", flag_exchange="p2p"),
            "ga": dict(collective="symm", flag_exchange="fused"),
            "ga-nccl": dict(collective="nccl", fuse=True),
            "bsp": dict(collective="symm", flag_exchange="fused", order="adaptive"),
            "nan_safe": dict(collective="symm", flag_exchange="fused", order="nan_safe"),
            "nccl-nansafe": dict(collective="nccl", nan_safe=True)}[variant]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    c = LARGE
    P = c["P"]
    init = torch.from_numpy(large_init(c["seed"], P)).to(dev)
    g = torch.zeros(P, device=dev)
    cfg = SelSyncConfig(delta=large_delta(variant), warmup=c["warmup"], smoothing=c["smoothing"],
                        momentum=c["momentum"], weight_decay=c["weight_decay"],
                        aggregation=large_aggregation(variant))
    step = SelSyncStep(init, g, cfg, tile_elems=c["tile"], **opts)
    g = step.grads  # gradient aggregation over symmetric memory owns the gradient buffer
    for s in range(c["steps"]):
        g.copy_(torch.from_numpy(O.synthetic_grad32(c["seed"], rank, s, P)), non_blocking=True)
        if step.async_capable:
            step.step_async(c["lr"])
        else:
            step.step(c["lr"])
    step.synchronize()
    recs = step.records()
    np.savez(out / f"large_{variant}_rank{rank}.npz", decisions=np.array(step.decisions()),
             ewma=np.array([r["ewma"] for r in recs]), params=step.params.double().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "large":
    large_main()
elif __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "nan"):
    main()


NAN_MODES = {"symm-adaptive": dict(collective="symm", order="adaptive"),
             "symm-known": dict(collective="symm", order="adaptive"),  # warmup 8: the known-sync pass
             "symm-update-first": dict(collective="symm", order="update_first"),
             "symm-nansafe": dict(collective="symm", order="nan_safe"),
             "nccl": dict(collective="nccl"),
             "nccl-nansafe": dict(collective="nccl", nan_safe=True)}


def nan_main():
    """A NaN gradient on ONE rank must raise SignalError on EVERY rank (the
    error bit travels with the agreed word), must never reach another rank's
    parameters, and in the NaN-safe orders must leave every rank's
    parameters and momentum untouched (signal.py:67-68 raises before
    sgd_step, strategies.py:286 vs :383)."""
    mode, out = sys.argv[2], Path(sys.argv[3])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2307_07950_b200 import SignalError

    P = 40_000
    w = torch.from_numpy(np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)).to(dev)
    g = torch.zeros(P, device=dev)
    warmup = 8 if mode == "symm-known" else 1
    cfg = SelSyncConfig(delta=0.1, warmup=warmup, smoothing=0.5, momentum=0.9, weight_decay=4e-4)
    step = SelSyncStep(w, g, cfg, tile_elems=4096, **NAN_MODES[mode])
    g = step.grads
    for s in range(3):
        g.copy_(torch.from_numpy(O.synthetic_grad32(5, rank, s, P)))
        step.step(0.1)
    before = step.params.clone()
    mom = step.momentum.clone()
    g.copy_(torch.from_numpy(O.synthetic_grad32(5, rank, 3, P)))
    if rank == 1:
        g[P // 2 + 7] = float("nan")
    raised = False
    try:
        if step.async_capable:
            step.step_async(0.1)
            step.synchronize()
        else:
            step.step(0.1)
    except SignalError:
        raised = True
    torch.cuda.synchronize()
    np.savez(out / f"nan_{mode}_rank{rank}.npz", raised=np.array(raised),
             finite=np.array(bool(torch.isfinite(step.params).all())),
             unchanged=np.array(bool(torch.equal(step.params, before) and torch.equal(step.momentum, mom))))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "nan":
    nan_main()
