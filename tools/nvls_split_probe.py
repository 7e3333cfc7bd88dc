"""NVLink mean decomposition probe (torchrun, 4 ranks; tooling, not product).

Times the modes of tools/nvls_split_probe.cu on a 400 MB symmetric fp32
buffer: the product NVLS mean, its two halves alone (ld_reduce only,
multicast store only), the P2P two-shot, NVLS + P2P splits of the shard, and
ld_reduce + P2P stores. Prints the time and the bytes per link direction
(the busier direction) / time for each.

  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
       -o tools/_nvls_split_probe.so tools/nvls_split_probe.cu
  torchrun --nproc-per-node 4 tools/nvls_split_probe.py [P]
"""
import ctypes
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

P = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
lib = ctypes.CDLL(str(Path(__file__).resolve().parent / "_nvls_split_probe.so"))
lib.probe_launch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                             ctypes.c_long, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                             ctypes.c_int, ctypes.c_int, ctypes.c_void_p]

buf = symm_mem.empty(P, dtype=torch.float32, device=dev)
hdl = symm_mem.rendezvous(buf, dist.group.WORLD)
buf.normal_()
ptrs = (ctypes.c_void_p * 8)(*([int(p) for p in hdl.buffer_ptrs] + [0] * (8 - world)))
mc = int(hdl.multicast_ptr)
nvec = P // 4
per = (nvec + world - 1) // world
v0 = min(per * rank, nvec)
v1 = min(v0 + per, nvec)
S = 4 * P
stream = torch.cuda.current_stream().cuda_stream


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
        # every rank's pass ends before the next one reads (as between steps)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def launch(mode, grid=296, block=512, split_vec=0, nvls_blocks=0):
    rc = lib.probe_launch(ptrs, mc, rank, world, v0, v1, split_vec, nvls_blocks, mode, 1.0 / world, grid, block,
                          stream)
    assert rc == 0, rc


def report(name, ms, dir_bytes):
    if rank == 0:
        busbw = S / (ms * 1e-3) / 1e9 * 2 * (world - 1) / world
        print(f"{name:44s} {ms * 1e3:8.1f} us  busbw {busbw:6.1f}  "
              f"{dir_bytes / S:.3f} S per dir -> {dir_bytes / (ms * 1e-3) / 1e9:6.1f} GB/s per dir", flush=True)


n = world
report("NVLS mean (ld_reduce + mc st)", timeit(lambda: launch(0)), S * (1 + 1 / n))
for g in (148, 592):
    report(f"NVLS mean grid {g}", timeit(lambda: launch(0, grid=g)), S * (1 + 1 / n))
report("ld_reduce only (local st)", timeit(lambda: launch(1)), S)
report("mc st only (local ld)", timeit(lambda: launch(2)), S)
report("P2P two-shot", timeit(lambda: launch(3)), S * 2 * (n - 1) / n)
report("ld_reduce + P2P st", timeit(lambda: launch(5)), S + S * (n - 1) / n)
for f in (0.1, 0.2, 0.3, 0.4, 0.5):
    nv = v1 - v0
    split = int(nv * (1 - f)) // 4 * 4
    cost_n, cost_p = (1 - f) * (1 + 1 / n), f * 2 * (n - 1) / n
    for share in (cost_n / (cost_n + cost_p), 1 - f):
        nb = max(1, min(295, round(296 * share)))
        report(f"split P2P {f:.1f}, NVLS blocks {nb}",
               timeit(lambda: launch(4, split_vec=split, nvls_blocks=nb)),
               S * ((1 - f) * (1 + 1 / n) + f * 2 * (n - 1) / n))
dist.barrier(device_ids=[local])
dist.destroy_process_group()
