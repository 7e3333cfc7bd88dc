"""Reproduce device-exchange timeouts: small P, each order, blocking steps."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.errors import TransportError  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
for P in (1002, 70000):
    for order in ("update_first", "norm_first"):
        for delta in (0.0, 1e9):
            w = torch.randn(P, device=dev)
            g = torch.randn(P, device=dev)
            st = SelSyncStep(w, g, SelSyncConfig(delta=delta, warmup=1), order=order, timeout_s=3.0)
            res = "ok"
            for s in range(6):
                try:
                    st.step(0.01)
                except TransportError as e:
                    res = f"timeout at step {s}: seq={int(st.symm.seq.item())} epoch={int(st.symm.epoch.item())} " \
                          f"pred={float(st.symm.predictor.item()):.2f}"
                    break
            out = [None] * world
            dist.all_gather_object(out, res)
            if rank == 0:
                print(f"P={P} order={order} delta={delta}: {out}", flush=True)
            dist.barrier(device_ids=[local])
dist.destroy_process_group()
