"""Tuning sweep of the streaming kernels at P=100M (each variant in a fresh
process; the choice is cached per process):
  SS_SGD_VARIANT "<cache policy><unroll>" for K3/K13 (0 = library default),
  SS_NORM_UNROLL for K1."""
import os
import subprocess
import sys

CODE = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2307_07950_b200 import kernels as K
P = 100_000_000
which = sys.argv[1]
dev = torch.device("cuda:0")
w = torch.randn(P, device=dev); g = torch.randn(P, device=dev); m = torch.zeros(P, device=dev)
sig = K.DeviceSignal(dev, 0.05, 1); ws = K.Workspace(dev); out = torch.empty(1, dtype=torch.float64, device=dev)
fns = {
  "k13_mom": (lambda: K.update_norm_signal_(w, g, m, sig, ws, lr=1e-6, delta=0.1, momentum=0.9, weight_decay=1e-4), 20),
  "k13_plain": (lambda: K.update_norm_signal_(w, g, None, sig, ws, lr=1e-6, delta=0.1), 12),
  "k3_mom": (lambda: K.sgd_update_(w, g, m, lr=1e-6, momentum=0.9, weight_decay=1e-4), 20),
  "k1": (lambda: K.norm_sq(g, out, ws), 4),
}
f, bpe = fns[which]
for _ in range(5): f()
torch.cuda.synchronize()
ts = []
for rep in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 20)
t = sorted(ts)[2]
print(f"{t*1e3:8.1f} us  {bpe*P/(t*1e-3)/1e9:7.1f} GB/s")
'''
plan = [("k13_mom", "SS_SGD_VARIANT", ["0", "2", "4", "11", "21", "31"]),
        ("k13_plain", "SS_SGD_VARIANT", ["0", "2", "4", "11", "21", "31"]),
        ("k3_mom", "SS_SGD_VARIANT", ["0", "2", "11", "21"]),
        ("k1", "SS_NORM_UNROLL", ["1", "2", "4", "8"])]
for which, var, vals in plan:
    for v in vals:
        out = subprocess.run([sys.executable, "-c", CODE, which], env={**os.environ, var: v},
                             capture_output=True, text=True)
        print(f"{which:10s} {var}={v:>3}: {out.stdout.strip()} {out.stderr.strip()[-200:]}", flush=True)
