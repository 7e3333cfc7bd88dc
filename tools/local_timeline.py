"""Where does a local step's time go at N > 1 (update-first order)? Device
timestamps of: step kernel start, vote posted (last block), all votes in.
Args: P, steps enqueued back to back per sample (marks are of the last one;
the event time is per step)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
B2B = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # steps enqueued back to back per sample
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
w = torch.randn(P, device=dev)
g = torch.randn(P, device=dev)
st = SelSyncStep(w, g, SelSyncConfig(delta=1e9, warmup=1, momentum=0.9, weight_decay=4e-4), order="update_first")
for _ in range(10):
    st.step_async(0.001)
st.synchronize()
tl = st.symm.enable_timeline(16)
rows = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(B2B):
        st.step_async(0.001)
    b.record()
    st.synchronize()
    mk = tl.cpu().numpy()[4 * 16:]
    rows.append(((mk[1] - mk[0]) / 1e3, (mk[2] - mk[1]) / 1e3, a.elapsed_time(b) * 1e3 / B2B, mk[0], mk[1]))
r = np.array(rows)
txt = (f"rank {rank}: start->vote posted {r[:,0].mean():.1f} us, vote wait {r[:,1].mean():.1f} us "
       f"(max {r[:,1].max():.1f}), event step {r[:,2].mean():.1f} us")
allt = [None] * world
dist.all_gather_object(allt, (txt, r[:, 3].tolist(), r[:, 4].tolist()))
if rank == 0:
    for t, _, _ in allt:
        print(t)
    starts = np.array([x[1] for x in allt]); posts = np.array([x[2] for x in allt])
    print("start skew across ranks (us): mean", ((starts.max(0) - starts.min(0)) / 1e3).mean().round(1),
          " vote-post skew:", ((posts.max(0) - posts.min(0)) / 1e3).mean().round(1))
dist.barrier(device_ids=[local])
dist.destroy_process_group()
