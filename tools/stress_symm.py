"""Stress of the device-side exchange: replay the n4_mixed golden case through
each step order with back-to-back async steps and pinned H2D copies (the
scenario that exposed the single-buffered vote slots); report timeouts."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from conftest import _load_cases  # noqa: E402
from oracle import selsync_oracle as O  # noqa: E402
from paper_2307_07950_b200 import SelSyncConfig  # noqa: E402
from paper_2307_07950_b200.errors import TransportError  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
c = _load_cases()["n4_mixed"]
P = c["P"]
variants = [(o, True, True, pin) for o in ("update_first", "norm_first", "adaptive") for pin in (False, True)]
host = [torch.from_numpy(O.synthetic_grad32(c["grad_seed"], rank, s, P)).pin_memory() for s in range(c["steps"])]
for order, alt, bc, pin in variants:
    init = torch.tensor(c["init"], dtype=torch.float32, device=dev)
    if bc and rank != 0:
        init = torch.full((P,), 7.0, device=dev)
    g = torch.zeros(P, device=dev)
    cfg = SelSyncConfig(delta=c["delta"], warmup=c["warmup"], smoothing=c["smoothing"])
    st = SelSyncStep(init, g, cfg, order=order, timeout_s=3.0)
    log = []
    res = "ok"
    for s in range(c["steps"]):
        if pin:
            g.copy_(host[s], non_blocking=True)
            pred = -1.0
        else:
            g.copy_(torch.from_numpy(O.synthetic_grad32(c["grad_seed"], rank, s, P)))
            pred = float(st.symm.predictor[int(st.symm.predictor[4].item()) & 3].item())
        try:
            if alt and s % 2:
                st.step_async(c["lr"])
                d = "async"
            else:
                d = st.step(c["lr"])
        except TransportError:
            res = f"timeout at step {s} (pred before {pred:.3f}) log tail {log[-4:]}"
            break
        log.append((s, d[0], round(pred, 3)))
    if res == "ok":
        try:
            st.synchronize()
        except TransportError:
            res = "timeout found at synchronize()"
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        print(f"order={order} alternate={alt} bcast_init={bc} pinned={pin}:", flush=True)
        for r, o in enumerate(out):
            print(f"   rank {r}: {o}", flush=True)
    dist.barrier(device_ids=[local])
dist.destroy_process_group()
