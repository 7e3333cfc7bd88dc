"""Host-to-device rates of a 400 MB fp32 gradient in pinned host memory
(tooling): one copy-engine cudaMemcpyAsync, the copy split over 2 / 4 streams,
SM loads straight from the host pointer (zero-copy kernel, several grids), and
the K13 step reading its gradient straight from the host pointer through a
prepared step plan."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
P = 100_000_000
dev = torch.device("cuda", 0)
host = torch.randn(P).pin_memory()
d = torch.empty(P, device=dev)
lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "_h2d_probe.so"))
lib.pull_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]


def t(fn, iters=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    return ms, 4 * P / (ms * 1e-3) / 1e9


print("copy engine, one memcpy: %.3f ms %.1f GB/s" % t(lambda: d.copy_(host, non_blocking=True)))
for k in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    cur = torch.cuda.current_stream()
    hs, ds = host.chunk(k), d.chunk(k)

    def split():
        for s, h_, d_ in zip(streams, hs, ds):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d_.copy_(h_, non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    print(f"copy engines, {k} streams: %.3f ms %.1f GB/s" % t(split))
st = torch.cuda.current_stream().cuda_stream
for grid in (148, 296, 592, 1184):
    for block in (256, 512):
        print(f"zero-copy kernel grid {grid} x {block}: %.3f ms %.1f GB/s" % t(
            lambda: lib.pull_launch(d.data_ptr(), host.data_ptr(), P // 4, grid, block, st)))
# the K13 step with its gradient read straight from pinned host memory (plan path)
from paper_2307_07950_b200 import _native as N  # noqa: E402
from paper_2307_07950_b200 import kernels as K  # noqa: E402
w = torch.randn(P, device=dev) * 0.01
m = torch.zeros(P, device=dev)
sig = K.DeviceSignal(dev, 1.0, 1, 64)
ws = K.Workspace(dev)
desc = N.RankStepC(w.data_ptr(), d.data_ptr(), m.data_ptr(), P, 0.9, 0.0, 4e-4, 0, sig.state.data_ptr(), 0.3,
                   sig.word.data_ptr(), sig.trace.data_ptr(), 64, 0, None, ws.ptr)
plan = N.StepPlanC()
N.check(N.LIB.ss_step_plan_init(ctypes.addressof(plan), ctypes.addressof(desc), 0))
print("K13 step, g in HBM: %.3f ms" % t(lambda: N.LIB.ss_step_plan_launch(ctypes.addressof(plan), d.data_ptr(), 0.01, 0, st))[0])
print("K13 step, g read from pinned host memory: %.3f ms (%.1f GB/s of PCIe)" % t(
    lambda: N.LIB.ss_step_plan_launch(ctypes.addressof(plan), host.data_ptr(), 0.01, 0, st)))
print("copy + K13 step: %.3f ms" % t(lambda: (d.copy_(host, non_blocking=True),
                                               N.LIB.ss_step_plan_launch(ctypes.addressof(plan), d.data_ptr(), 0.01, 0, st)))[0])
