"""Back-to-back async steps (no host sync): does the next step ever overlap the
previous step's device-launched mean?"""
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
for P in (1002, 4_000_000):
    for order in ("update_first", "norm_first"):
        w = torch.full((P,), 1.0, device=dev)
        g = torch.zeros(P, device=dev)
        st = SelSyncStep(w, g, SelSyncConfig(delta=0.0, warmup=1), order=order, timeout_s=3.0)
        # each rank's gradient is rank-dependent: after a sync step every replica
        # must equal the mean exactly (w - lr * mean(g)), whatever the overlap
        g.fill_(float(rank))
        res = "ok"
        for s in range(40):
            st.step_async(0.01)
        try:
            st.synchronize()
            want = 1.0 - 40 * 0.01 * (world - 1) / 2.0
            err = float((st.params - want).abs().max())
            if err > 1e-4:
                res = f"WRONG params: max err {err:.3g}"
        except TransportError:
            res = f"timeout (seq={int(st.symm.seq.item())})"
        out = [None] * world
        dist.all_gather_object(out, res)
        if rank == 0:
            print(f"P={P} order={order}: {out}", flush=True)
        dist.barrier(device_ids=[local])
dist.destroy_process_group()
