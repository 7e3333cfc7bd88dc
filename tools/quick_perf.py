"""Kernel-level bandwidth probe (CUDA events, inputs >> L2). Not the bench."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import kernels as K  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda:0")
w = torch.randn(P, device=dev)
g = torch.randn(P, device=dev)
m = torch.zeros(P, device=dev)
sig = K.DeviceSignal(dev, 0.05, 1)
ws = K.Workspace(dev)
out = torch.empty(1, dtype=torch.float64, device=dev)


def bench(name, fn, nbytes, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    med = ts[len(ts) // 2]
    print(f"{name:28s} median {med*1e3:8.1f} us  {nbytes / (med * 1e-3) / 1e9:8.1f} GB/s  (min {ts[0]*1e3:.1f} us)")


bench("K1 norm", lambda: K.norm_sq(g, out, ws), 4 * P)
bench("K1+K2 norm_signal", lambda: K.norm_signal(g, sig, 0.1, ws), 4 * P)
bench("K3 sgd plain", lambda: K.sgd_update_(w, g, None, lr=1e-6), 12 * P)
bench("K3 sgd mom+wd", lambda: K.sgd_update_(w, g, m, lr=1e-6, momentum=0.9, weight_decay=1e-4), 20 * P)
bench("K13 fused plain", lambda: K.update_norm_signal_(w, g, None, sig, ws, lr=1e-6, delta=0.1), 12 * P)
bench("K13 fused mom+wd", lambda: K.update_norm_signal_(w, g, m, sig, ws, lr=1e-6, delta=0.1, momentum=0.9, weight_decay=1e-4), 20 * P)
bench("torch copy (ref)", lambda: w.copy_(g), 8 * P)
bench("torch dot fp32", lambda: torch.dot(g, g), 4 * P)
