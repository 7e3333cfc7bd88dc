"""The one-launch SelSync step kernel on ONE GPU (world-1 symmetric memory),
so ncu can profile it (ncu only runs single-GPU commands here).

  python tools/step_kernel_solo.py ORDER MODE [P]
    ORDER: update_first | norm_first     MODE: local (delta 1e9) | sync (delta 0)

At world 1 the vote exchange is with itself and the "mean" of a sync step is
a copy of the own buffer through the same NVLink code path (P2P width 1), so
the update / norm sweep / ticket machinery is what gets measured."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

order, mode = sys.argv[1], sys.argv[2]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000_000
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
w = torch.randn(P, device=dev) * 0.05
g = torch.randn(P, device=dev)
cfg = SelSyncConfig(delta=1e9 if mode == "local" else 0.0, warmup=1, momentum=0.9, weight_decay=4e-4)
st = SelSyncStep(w, g, cfg, collective="symm", order=order)
assert st.collective == "symm" and st.flag_exchange == "fused"
for _ in range(5):
    st.step_async(0.01)
st.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
graph = st.capture(0.01) if os.environ.get("GRAPH") else None  # launch-bound sizes: one graph per step
a.record()
for _ in range(n):
    if graph is not None:
        graph.replay()
    else:
        st.step_async(0.01)
b.record()
st.synchronize()
ms = a.elapsed_time(b) / n
nbytes = (24 if order == "norm_first" else 20) * P
print(f"order={order} mode={mode} P={P:,}: {ms * 1e3:.1f} us/step, {nbytes / (ms * 1e-3) / 1e9:.0f} GB/s "
      f"algorithmic (update{' + norm sweep' if order == 'norm_first' else ''}; sync adds a self-copy of 8P)",
      flush=True)
dist.destroy_process_group()
