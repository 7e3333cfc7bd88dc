"""Timeline of the overlapped (norm-first) sync step: per-ticket timestamps
from the device, summarised per rank (torchrun, one rank per GPU).
Args: P, tile, mode (known | up | down | up-early)."""
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
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
w = torch.randn(P, device=dev)
g = torch.randn(P, device=dev)
# mode: known (delta = 0: the known-sync pass) | up / down (delta 0.3, smoothing 1:
# a sync step on an upward / downward jump of ||g||^2 after local steps) |
# up-early (the same upward step with the opt-in exact early vote)
mode = sys.argv[3] if len(sys.argv) > 3 else "known"
if mode == "known":
    cfg = SelSyncConfig(delta=0.0, warmup=1, momentum=0.9, weight_decay=4e-4)
else:
    cfg = SelSyncConfig(delta=0.3, warmup=1, smoothing=1.0, momentum=0.9, weight_decay=4e-4)
st = SelSyncStep(w, g, cfg, order="norm_first", tile_elems=tile, early_vote=mode == "up-early")
if mode == "down":
    g.mul_(1.5)
for _ in range(5):
    st.step_async(0.01)
st.synchronize()
if mode in ("up", "up-early"):
    g.mul_(1.5)
elif mode == "down":
    g.div_(1.5)
cap = 8 * (P // tile + 64)
tl = st.symm.enable_timeline(cap)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
st.step_async(0.01)
b.record()
st.synchronize()
ms = a.elapsed_time(b)
raw = tl.cpu().numpy()
marks = raw[4 * cap:]
ev = raw[: 4 * cap].reshape(-1, 4)
ev = ev[ev[:, 1] > 0]
kind = ev[:, 0] >> 48
t0 = ev[:, 1].min()
out = {}
for name, kk in (("update", 0), ("mean", 1)):
    e = ev[kind == kk]
    if len(e) == 0:
        continue
    wait = (e[:, 2] - e[:, 1]) / 1e3
    run = (e[:, 3] - e[:, 2]) / 1e3
    out[name] = (len(e), wait.mean(), run.mean(), (e[:, 1].min() - t0) / 1e3, (e[:, 3].max() - t0) / 1e3,
                 np.percentile(run, 90))
span = (ev[:, 3].max() - t0) / 1e3
m0 = marks[0]
dec = st.decisions()[-1]
lines = [f"rank {rank} [{mode}, decision {dec}]: step {ms*1e3:.0f} us (events), overlapped kernel span {span:.0f} us",
         "   vote posted {:.0f} us; early sync posted {}; first ticket {:.0f}; last arrival {:.0f}; "
         "end barrier done {:.0f} us".format(
             (marks[1] - m0) / 1e3, f"{(marks[3] - m0) / 1e3:.0f} us" if marks[3] > m0 else "-", (t0 - m0) / 1e3,
             (marks[4] - m0) / 1e3, (marks[5] - m0) / 1e3)]
for name, (n, wt, rn, first, last, p90) in out.items():
    lines.append(f"   {name:6s} tasks {n:5d}  wait {wt:7.1f} us  run {rn:7.1f} us (p90 {p90:.1f})  "
                 f"first start {first:7.0f} us  last end {last:7.0f} us")
# concurrency: how many mean tasks were running over time
m = ev[kind == 1]
if len(m):
    grid = np.linspace(0, span, 20)
    conc = [int(((m[:, 2] - t0) / 1e3 <= x).sum() - ((m[:, 3] - t0) / 1e3 <= x).sum()) for x in grid]
    upd = ev[kind == 0]
    concu = [int(((upd[:, 1] - t0) / 1e3 <= x).sum() - ((upd[:, 3] - t0) / 1e3 <= x).sum()) for x in grid]
    lines.append("   running mean tasks over time:   " + " ".join(f"{c:3d}" for c in conc))
    lines.append("   running update tasks over time: " + " ".join(f"{c:3d}" for c in concu))
txt = "\n".join(lines)
all_txt = [None] * world
dist.all_gather_object(all_txt, txt)
if rank == 0:
    print("\n".join(all_txt), flush=True)
dist.barrier(device_ids=[local])
dist.destroy_process_group()
