"""Parameter-averaging bandwidth probe (torchrun, one rank per GPU).

Times, on the same 4P-byte fp32 buffer: our device-conditional exchange
kernel (ss_symm_sync_f32, word forced to sync) on the NVLS multicast path
and on the P2P two-shot path, NCCL allreduce-AVG, and torch's symmetric-
memory all-reduces (reference points). busbw = (4P / t) * 2(N-1)/N.
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_07950_b200 import kernels as K  # noqa: E402
from paper_2307_07950_b200.collectives import RankGroup, SymmetricParams  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
ITERS = 20
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = RankGroup()


def timeit(fn, iters=ITERS):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return comm.max_float(a.elapsed_time(b) / iters, dev)


def report(name, ms):
    algbw = 4 * P / (ms * 1e-3) / 1e9
    busbw = algbw * 2 * (world - 1) / world
    if rank == 0:
        print(f"N={world} P={P:,} {name:34s} {ms * 1e3:9.1f} us  busbw {busbw:7.1f} GB/s", flush=True)


ws = K.Workspace(dev)
word = torch.ones(1, dtype=torch.int32, device=dev)
for mc in (() if os.environ.get("SYMM_NCCL_ONLY") else (True, False)):  # explicit choice per path
    sp = SymmetricParams(P, dev, comm, use_multicast=mc)
    sp.buf.normal_()
    if rank == 0:
        print(f"multicast requested={mc} available={sp.multicast}", flush=True)
    if mc and not sp.multicast:
        continue
    ms = timeit(lambda: sp.sync_(word, ws.ptr, exchange=False, stream=torch.cuda.current_stream().cuda_stream))
    sp.check()
    report(f"ss_symm_sync {'NVLS multimem' if sp.multicast else 'P2P two-shot'}", ms)
    word0 = torch.zeros(1, dtype=torch.int32, device=dev)
    ms = timeit(lambda: sp.sync_(word0, ws.ptr, exchange=False, stream=torch.cuda.current_stream().cuda_stream), 200)
    if rank == 0:
        print(f"    local step (word=0, early exit): {ms * 1e3:.1f} us", flush=True)
    w2 = torch.zeros(1, dtype=torch.int32, device=dev)
    ms = timeit(lambda: (w2.fill_(1), sp.sync_(w2, ws.ptr, exchange=True, stream=torch.cuda.current_stream().cuda_stream)), 200)
    if rank == 0:
        print(f"    p2p flag exchange + sync: {ms * 1e3:.1f} us", flush=True)
    w3 = torch.zeros(1, dtype=torch.int32, device=dev)
    ms = timeit(lambda: (w3.zero_(), sp.sync_(w3, ws.ptr, exchange=True, stream=torch.cuda.current_stream().cuda_stream)), 200)
    if rank == 0:
        print(f"    p2p flag exchange, local: {ms * 1e3:.1f} us", flush=True)

if os.environ.get("SYMM_ONLY"):
    dist.barrier(device_ids=[local])
    dist.destroy_process_group()
    sys.exit(0)
buf = torch.randn(P, device=dev)
report("nccl all_reduce AVG", timeit(lambda: dist.all_reduce(buf, op=dist.ReduceOp.AVG)))
report("nccl all_reduce SUM", timeit(lambda: dist.all_reduce(buf, op=dist.ReduceOp.SUM)))
wd = torch.ones(1, dtype=torch.int32, device=dev)
ms = timeit(lambda: dist.all_reduce(wd, op=dist.ReduceOp.MAX), 200)
if rank == 0:
    print(f"    nccl allreduce-MAX int32[1]: {ms * 1e3:.1f} us", flush=True)
try:
    import torch.distributed._symmetric_memory as symm_mem

    t = symm_mem.empty(P, dtype=torch.float32, device=dev).normal_()
    symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    for op in ("multimem_all_reduce_", "two_shot_all_reduce_"):
        fn = getattr(torch.ops.symm_mem, op, None)
        if fn is None:
            continue
        try:
            report(f"torch symm_mem.{op}", timeit(lambda: fn(t, "sum", dist.group.WORLD.group_name)))
        except Exception as exc:  # noqa: BLE001
            if rank == 0:
                print(f"torch symm_mem.{op}: {type(exc).__name__}: {str(exc)[:200]}")
except Exception as exc:  # noqa: BLE001
    if rank == 0:
        print("torch symm_mem unavailable:", exc)
dist.barrier(device_ids=[local])
dist.destroy_process_group()
