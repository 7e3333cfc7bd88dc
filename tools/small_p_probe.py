"""Small-P local step at N ranks (torchrun): per-step time of the one-launch
step (delta = 1e9: every step after the warmup one is local) for a few grid
caps (the group's max_blocks), eager back-to-back launches and CUDA-graph
replays; max over ranks, CUDA events. Args: P list (comma-separated)."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.collectives import RankGroup  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

Ps = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1000000,4000000").split(",")]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = RankGroup()
ITERS = 300


def time_it(fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    comm.barrier(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(ITERS):
        fn()
    b.record()
    torch.cuda.synchronize()
    return comm.max_float(a.elapsed_time(b) * 1e3 / ITERS, dev)


for P in Ps:
    w = torch.randn(P, device=dev)
    g = torch.randn(P, device=dev) * 1e-3
    for order in os.environ.get("ORDERS", "update_first,adaptive").split(","):
        for mb in [int(x) for x in os.environ.get("MAX_BLOCKS", "0,296,148,74").split(",")]:
            # SYNC=1: delta = 0, every step a (known-sync pass) sync step
            cfg = SelSyncConfig(delta=0.0 if os.environ.get("SYNC") == "1" else 1e9, warmup=1, momentum=0.9,
                                weight_decay=4e-4)
            st = SelSyncStep(w.clone(), g, cfg, group=comm, order=order, max_blocks=mb)
            st.step_async(1e-3)
            eager = time_it(lambda: st.step_async(1e-3))
            graph = st.capture(1e-3)
            replay = time_it(graph.replay)
            st.synchronize()
            if rank == 0:
                print(f"{os.environ.get('TAG', '')} N={world} P={P:>9,} {order:12s} max_blocks={mb:4d}: eager {eager:6.1f} us  "
                      f"graph {replay:6.1f} us", flush=True)
dist.barrier(device_ids=[local])
dist.destroy_process_group()
