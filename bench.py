#!/usr/bin/env python
"""SelSync hot-path benchmark on B200 (contract: one JSON line from rank 0).

Workload (BASELINE.json configs[4] at the north_star's target size): one
SelSync step per iteration over a flattened fp32 model of P = 100M
parameters, SGD with momentum 0.9 and weight decay 4e-4 (the paper's
ResNet-101 optimizer), synthetic gradients already resident
in HBM. A step is the whole hot path:

  K13+K2 (fused update + ||g||^2 + EWMA/Delta/decide)
  -> C1 flag-word MAX over ranks
  -> C2 mean of the 400 MB parameter buffer on sync steps.

At N = 1 that is one K13 launch. At N > 1 (default --collective symm
--flag-exchange fused) it is ONE launch of the symmetric-memory step kernel
(ss_step_symm_f32): C1 as a seq-tagged NVLink P2P vote and C2 as an NVLS
multicast (N >= 4) or P2P two-shot (N = 2) mean with 1/N in registers,
overlapped tile by tile with the update in the norm-first order.
``--collective nccl`` is the literal north_star variant (NCCL allreduce-MAX
of an int32 word, NCCL allreduce-AVG of the buffer) kept for comparison.

The headline ``value`` is steps/s of the whole job under a decision mix with
exactly 50% sync steps (gradient ring with scales [1, 1, 1.5, 1.5], EWMA
smoothing 1.0, delta 0.3: Delta alternates 0 / >= 0.55); the forced
all-local (delta = 1e9) and all-sync (delta = 0) rates are measured in the
same run under ``modes``. ``e2e`` is the same step through the public API
with the gradient copied from pinned host memory every step and the
decision row read back. ``cpu_baseline`` / ``--impl reference`` time the
reference's float64 CPU path (oracle/cpu_path.py) on this host.

Run: python bench.py [--gpus N --steps K --warmup W]; N > 1 under torchrun.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SelSync steps/s and hot-path GB/s vs HBM/NVLink roofline"
FALLBACK_HBM_GBS = 6650.0
NVLINK_NOMINAL_GBS = 900.0
NVLINK_ALLREDUCE_MEASURED_GBS = 725.0  # B200_PROFILING.md: 8-rank all-reduce busbw at 1 GiB
MIX_SCALES = [1.0, 1.0, 1.5, 1.5]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--P", type=int, default=100_000_000)
    ap.add_argument("--workload", default="microbench", choices=["microbench", "resnet101", "vgg11", "transformer"],
                    help="microbench: the hot path on resident synthetic gradients (headline); model "
                         "workloads add stock PyTorch fwd/bwd of BASELINE configs 1-3")
    ap.add_argument("--delta", type=float, default=0.3, help="delta for model workloads")
    ap.add_argument("--graph", action="store_true",
                    help="model workloads: capture fwd + bwd + SelSync step in one CUDA graph; microbench: "
                         "replay captured steps (launch-bound small P)")
    ap.add_argument("--graph-steps", type=int, default=1,
                    help="microbench --graph: consecutive steps per captured graph (the gradient ring in order; "
                         "remainders replay one-step graphs)")
    ap.add_argument("--sel-warmup", type=int, default=25, help="EWMA window / warmup for model workloads")
    ap.add_argument("--momentum", type=float, default=0.9)
    ap.add_argument("--weight-decay", type=float, default=4e-4)
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--no-fuse", action="store_true", help="pre-scale order (K1+K2, C1, K3*1/N, SUM)")
    ap.add_argument("--collective", default="symm", choices=["symm", "nccl"],
                    help="C2 back end at N > 1: device-conditional symmetric-memory kernel or host-branch NCCL")
    ap.add_argument("--flag-exchange", default="fused", choices=["fused", "p2p", "nccl"],
                    help="fused: the whole step in one cooperative launch (symm only)")
    ap.add_argument("--tile", type=int, default=None,
                    help="elements per tile of the overlapped sync step (default: 4096 up to 2M params, else 16384)")
    ap.add_argument("--order", default="auto", choices=["auto", "update_first", "norm_first", "adaptive", "nan_safe"],
                    help="one-launch step order (flag-exchange fused): norm_first overlaps update and mean")
    ap.add_argument("--early-vote", action="store_true",
                    help="norm-first orders: the exact early vote (opt-in; A/B of the mean's start)")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="no per-launch CUDA events (latency-bound small P: the events themselves cost "
                         "a few us per step); the roofline then uses the whole local step time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-replay", action="store_true", help="skip the replayed golden decision patterns")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    return ap.parse_args()


def cpu_model() -> str:
    """The host CPU's model name (the baseline's hardware, stated with its core count)."""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bind_host_to_gpu(index: int):
    """Bind this process to the CPUs NVML lists as closest to GPU `index` (its
    NUMA node) while the e2e arm allocates its pinned host buffers, so its H2D
    copies read memory local to the GPU. SS_BENCH_NUMA=0 skips it. Returns
    the CPU count bound to, or None."""
    if os.environ.get("SS_BENCH_NUMA", "1") == "0":
        return None
    try:
        import pynvml
        import torch

        pr = torch.cuda.get_device_properties(index)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [64 * w + b for w, word in enumerate(words) for b in range(64) if (word >> b) & 1]
        cpus = [c for c in cpus if c < os.cpu_count()]
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return len(cpus)
    except Exception:  # no NVML / no affinity info: leave the scheduler alone
        return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the GPU is busy."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples = []
        self.ok = False
        self.period = period_s
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # no NVML: report it, never block the bench
            self.err = str(exc)
        self._stop = threading.Event()
        self._t = None

    def _reasons(self):
        nv = self.nv
        fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        return int(fn(self.h))

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                     self._reasons()))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._stop.clear()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t is not None:
            self._stop.set()
            self._t.join()
            self._t = None

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": f"nvml unavailable: {self.err}"}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = sorted(s for s, _ in self.samples)
        bits = 0
        for _, r in self.samples:
            bits |= r
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if bits & b], "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU arm


def cpu_run(n_workers, P, steps, warmup, args, budget_s):
    """Time the reference's CPU path (oracle/cpu_path.py) on a bounded sample:
    P_sample parameters per worker chosen so the run fits the budget, time
    scaled linearly to P (every op on the path is a linear pass over P)."""
    import numpy as np  # noqa: F401

    from oracle.cpu_path import CpuSelSync

    def make(p):
        return CpuSelSync(n_workers, p, delta=0.3, warmup=1, smoothing=1.0, momentum=args.momentum,
                          weight_decay=args.weight_decay, sync_pattern=MIX_SCALES, grad_ring=4)

    probe_p = min(P, 2_000_000)
    probe = make(probe_p)
    probe.time_steps(2, args.lr)
    t_probe = probe.time_steps(4, args.lr) / 4
    probe.close()
    per_elem = t_probe / probe_p
    total_steps = steps + warmup
    p_sample = int(min(P, max(8_000_000, budget_s / max(total_steps, 1) / max(per_elem, 1e-15))))
    p_sample = min(p_sample, P)
    cpu = make(p_sample)
    cpu.time_steps(warmup, args.lr)
    syncs0 = cpu.syncs
    secs = cpu.time_steps(steps, args.lr)
    syncs = cpu.syncs - syncs0
    threads = cpu.threads
    cpu.close()
    per_step_full = secs / steps * (P / p_sample)
    return {
        "value": n_workers / per_step_full,
        "unit": "steps/s",
        "cores": threads,
        "host_cpus": os.cpu_count(),
        "cpu_model": cpu_model(),
        "kind": "port",
        "sample": (f"{steps} timed steps of the reference's float64 SelSync step (oracle/cpu_path.py: "
                   f"g@g, observe/decide, SGD+momentum+wd, flag OR, on sync f64 serialize + PS "
                   f"np.stack().mean + deserialize) for {n_workers} worker(s) at P_sample={p_sample:,} "
                   f"({syncs}/{steps} sync steps), vectors sliced over {threads} host threads, "
                   f"time scaled x{P / p_sample:.2f} to P={P:,}"),
        "sec_per_step_sample": secs / steps,
    }


def reference_arm(args, rank, world):
    if rank != 0:
        return
    budget = 150.0
    base = cpu_run(world, args.P, args.steps, args.warmup, args, budget)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": base["value"],
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * world / base["value"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp64",
        "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "host_cpus", "cpu_model", "kind", "sample")},
        "e2e": {"value": base["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    from paper_2307_07950_b200.collectives import resolve_order

    return {
        "workload": (f"selsync hot-path step, flattened fp32 model P={args.P:,} (BASELINE configs[4] "
                     f"microbench at the north_star 100M size), SGD momentum {args.momentum} wd "
                     f"{args.weight_decay}, 50% sync decision mix"),
        "P": args.P,
        "n_workers": world,
        "update_kernel": "K1+K2 then K3 with 1/N pre-scale" if args.no_fuse else "fused K13+K2",
        "collective": args.collective if world > 1 else "none (single rank)",
        "flag_exchange": args.flag_exchange if world > 1 else "none (single rank)",
        "step_order": (resolve_order(args.order, args.P, world) if world > 1 and args.flag_exchange == "fused"
                       else "update_first"),
        "early_vote": bool(world > 1 and args.order in ("norm_first", "adaptive") and args.early_vote),
        "decision_mix": {"sync_frac": 0.5, "grad_scales": MIX_SCALES, "smoothing": 1.0, "delta": 0.3,
                         "warmup": 1},
        "parallelism": (f"dp{world} (SelSync replicas; vote + mean over "
                        + ("NVLink symmetric memory" if args.collective == "symm" else "NCCL") + ")"
                        if world > 1 else "dp1 (single replica, no exchange)"),
        "value_counts": "worker-steps: N ranks x K steps / (max-over-ranks device time)",
        "l2": (f"inputs exceed L2: w, g, m = {12 * args.P / 1e9:.2f} GB per step vs 126 MB L2"
               if 12 * args.P > 126e6 else
               f"inputs fit in L2 ({12 * args.P / 1e6:.1f} MB, not flushed): a small-P sweep point, "
               "launch/latency-bound, not a bandwidth claim"),
        "launch": ((f"CUDA graphs of {args.graph_steps} consecutive steps (the gradient ring in order, "
                    "programmatic dependent launch between the step kernels inside a graph)"
                    if args.graph_steps > 1 else "one CUDA graph replay per step (captured per gradient buffer)")
                   if args.graph else "one host launch per step (programmatic dependent launch)"),
    }


# ----------------------------------------------------------------- GPU arm


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2307_07950_b200 import SelSyncConfig
    from paper_2307_07950_b200 import kernels as K
    from paper_2307_07950_b200.collectives import RankGroup, resolve_order
    from paper_2307_07950_b200.step import SelSyncStep

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = RankGroup()
    P = args.P
    hbm_peak, hbm_src = peaks()
    if args.workload != "microbench":
        return model_bench(args, dev, comm, rank, world, local, hbm_peak, hbm_src)

    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    w = (torch.rand(P, generator=gen, device=dev) - 0.5) * 0.1
    # gradient ring: steps k = 0..3 use scales [1, 1, 1.5, 1.5] -> ||g||^2 ratio 2.25
    lo = torch.randn(P, generator=gen, device=dev) * MIX_SCALES[0]
    hi = torch.randn(P, generator=gen, device=dev) * MIX_SCALES[2]
    grads_ring = [lo, lo.clone(), hi, hi.clone()]
    g = torch.empty(P, device=dev)
    mom = torch.zeros(P, device=dev)

    def make_step(delta, smoothing=1.0, events=True):
        """events: CUDA events around every launch (the per-kernel times of the
        roofline); the headline run goes without them, back to back."""
        cfg = SelSyncConfig(delta=delta, warmup=1, smoothing=smoothing, momentum=args.momentum,
                            weight_decay=args.weight_decay)
        st = SelSyncStep(w, g, cfg, momentum_buffer=mom, group=comm, fuse=not args.no_fuse,
                         collective=args.collective if world > 1 else None,
                         flag_exchange=(args.flag_exchange if args.collective == "symm" else "nccl"),
                         trace_capacity=1 << 14, profile=events and not (args.graph or args.no_kernel_events),
                         order=args.order, tile_elems=args.tile, early_vote=args.early_vote)
        return st

    captured = {}  # --graph: one CUDA graph per (step object, gradient buffer)

    copy_s = torch.cuda.Stream(dev)
    gbufs = []

    def run(step, n, host_ring=None, host_row=None, schedule=None, prefetch=False):
        """n steps. Device-resident inputs: step_async (no host round-trip) when
        the step branches on the device. host_ring: the public blocking API with
        an H2D copy of the step's gradient from pinned host memory and a D2H of
        the step's decision row inside every step. schedule: ring index per step
        (a replayed decision pattern) instead of the period-4 ring."""
        if host_ring is not None and prefetch:
            # the H2D of step i+1's gradient (side stream, second device buffer)
            # runs while step i computes; PCIe stays busy back to back
            cur = torch.cuda.current_stream()
            copy_s.wait_stream(cur)
            with torch.cuda.stream(copy_s):
                gbufs[0].copy_(host_ring[step.steps_done % 4], non_blocking=True)
            for i in range(n):
                k = step.steps_done % 4
                ready = torch.cuda.Event()
                ready.record(copy_s)
                if i + 1 < n:
                    with torch.cuda.stream(copy_s):
                        gbufs[(i + 1) % 2].copy_(host_ring[(k + 1) % 4], non_blocking=True)
                cur.wait_event(ready)
                step.grads = gbufs[i % 2]
                step.step(args.lr)
                r = (step.steps_done - 1) % step.signal.trace_capacity  # this step's trace row
                host_row.copy_(step.signal.trace[32 * r:32 * r + 32], non_blocking=True)
                cur.synchronize()
            return
        i = 0
        while i < n:
            i += 1
            k = step.steps_done % 4 if schedule is None else schedule[step.steps_done % len(schedule)]
            G = args.graph_steps
            if (args.graph and step.async_capable and step.steps_done > 0 and schedule is None and host_ring is None
                    and G > 1 and n - i + 1 >= G):
                graphs = captured.setdefault(id(step), {})
                if ("multi", k) not in graphs:
                    graphs[("multi", k)] = step.capture(args.lr, [grads_ring[(k + j) % 4] for j in range(G)])
                graphs[("multi", k)].replay()
                i += G - 1
                continue
            if host_ring is not None:
                step.grads = g
                g.copy_(host_ring[k], non_blocking=True)
                step.step(args.lr)
                r = (step.steps_done - 1) % step.signal.trace_capacity  # this step's trace row
                host_row.copy_(step.signal.trace[32 * r:32 * r + 32], non_blocking=True)
                torch.cuda.current_stream().synchronize()
            elif args.graph and step.async_capable and step.steps_done > 0:
                graphs = captured.setdefault(id(step), {})
                if k not in graphs:
                    step.grads = grads_ring[k]
                    graphs[k] = step.capture(args.lr)
                graphs[k].replay()
            else:
                step.grads = grads_ring[k]  # bind this step's resident gradient
                if step.async_capable:
                    step.step_async(args.lr)
                else:
                    step.step(args.lr)

    def timed(step, n, **kw):
        comm.barrier(dev)
        torch.cuda.synchronize()
        launches0 = K.LAUNCHES
        k0 = len(step.kernel_events)
        s0 = len(step.sync_events)
        d0 = step.steps_done
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(step, n, **kw)
        b.record()
        torch.cuda.synchronize()
        step.synchronize()
        comm.barrier(dev)
        ms = comm.max_float(a.elapsed_time(b), dev)
        kms = step.kernel_ms()[k0:]
        sms = step.sync_ms()[s0:]
        dec = step.decisions()[d0 - step.steps_done:]
        return dict(ms=ms, decisions=dec, kernel_ms=kms, sync_ms=sms,
                    launches=K.LAUNCHES - launches0)

    clocks = ClockSampler(local)
    # ---- headline: 50% sync mix, device-resident inputs
    failure = None
    if world > 1 and args.collective == "symm":
        # safety net: if symmetric memory cannot be set up or the device-side
        # exchange times out on this box, ALL ranks agree to measure the NCCL
        # back end instead of hanging or dying
        from paper_2307_07950_b200.errors import TransportError

        try:
            mixed = make_step(0.3, events=False)
            run(mixed, args.warmup)
            mixed.synchronize()
        except (TransportError, RuntimeError) as exc:
            failure = exc
        if comm.max_float(1.0 if failure is not None else 0.0, dev) > 0.0:
            print(f"bench: symmetric-memory path failed on some rank ({failure}); falling back to NCCL",
                  file=sys.stderr, flush=True)
            args.collective = "nccl"
            mixed = make_step(0.3, events=False)
            run(mixed, args.warmup)
    else:
        mixed = make_step(0.3, events=False)
        run(mixed, args.warmup)
    clocks.start()
    res = timed(mixed, args.steps)
    clocks.stop()
    # ---- forced modes
    modes = {}
    for name, delta in (("all_local", 1e9), ("all_sync", 0.0)):
        st = make_step(delta)
        run(st, max(3, args.warmup))
        modes[name] = timed(st, args.steps)
    # ---- non-periodic mixes: the reference's own golden decision traces replayed
    #      (sync <=> the gradient scale switches between 1.0 and 1.5: Delta >= 0.55)
    replays = {}
    if not args.no_replay:
        for case, sched in replay_schedules().items():
            st = make_step(0.3)
            run(st, max(3, args.warmup), schedule=sched)
            replays[case] = (timed(st, args.steps, schedule=sched), sched)
    # ---- C2 alone (NVLink roofline of the mean): ss_symm_sync_f32 with the word forced to sync
    c2 = None
    if world > 1 and args.collective == "symm":
        sp = mixed.symm
        one = torch.ones(1, dtype=torch.int32, device=dev)
        cs = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            sp.sync_(one, mixed.ws.ptr, exchange=False, stream=cs)
        torch.cuda.synchronize()
        comm.barrier(dev)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(5, min(args.steps, 50))
        ea.record()
        for _ in range(reps):
            sp.sync_(one, mixed.ws.ptr, exchange=False, stream=cs)
        eb.record()
        torch.cuda.synchronize()
        sp.check()
        t = comm.max_float(ea.elapsed_time(eb), dev) / reps
        algbw = 4 * P / (t * 1e-3) / 1e9
        busbw = algbw * 2 * (world - 1) / world
        c2 = {"kernel": f"ss_symm_sync_f32 ({'NVLS multimem' if sp.multicast else 'P2P two-shot'}), word forced to sync",
              "mean_ms": t, "nvlink": {
                  "busbw": busbw, "algbw": algbw, "unit": "GB/s", "peak_nominal": NVLINK_NOMINAL_GBS,
                  "frac_nominal": busbw / NVLINK_NOMINAL_GBS,
                  "ref_nccl_allreduce_busbw_1GiB_8gpu": NVLINK_ALLREDUCE_MEASURED_GBS,
                  "frac_of_ref": busbw / NVLINK_ALLREDUCE_MEASURED_GBS},
              "sync_step_overlap_note": ("with the adaptive order a sync step overlaps the update with this "
                                         "mean (modes.all_sync.ms_per_step)")}
    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # pinned host buffers on the GPU's own NUMA node (first touch under a
        # temporary CPU binding; the scheduler's full set is restored at once)
        all_cpus = os.sched_getaffinity(0)
        numa_cpus = bind_host_to_gpu(local)
        host_ring = [t.cpu().pin_memory() for t in grads_ring[:1] + grads_ring[2:3]]
        host_ring = [host_ring[0], host_ring[0], host_ring[1], host_ring[1]]
        row = torch.empty(32, dtype=torch.uint8, pin_memory=True)
        os.sched_setaffinity(0, all_cpus)
        gbufs[:] = [g, torch.empty_like(g)]
        st = make_step(0.3)
        run(st, max(3, args.warmup), host_ring=host_ring, host_row=row)
        e_serial = timed(st, args.steps, host_ring=host_ring, host_row=row)
        st = make_step(0.3)
        run(st, max(3, args.warmup), host_ring=host_ring, host_row=row, prefetch=True)
        e = timed(st, args.steps, host_ring=host_ring, host_row=row, prefetch=True)
        e2e = {"value": world * args.steps / (e["ms"] / 1e3), "unit": "steps/s",
               "h2d_bytes_per_step": 4 * P * world, "d2h_bytes_per_step": 32 * world,
               "ms_per_step": e["ms"] / args.steps,
               "h2d_gbs_per_rank": 4 * P * args.steps / (e["ms"] * 1e-3) / 1e9,
               "serial_value": world * args.steps / (e_serial["ms"] / 1e3),
               "host_cpus_bound": numa_cpus,
               "note": ("per step and rank: H2D of the fp32 gradient from pinned host memory, the "
                        "SelSync step (public blocking API), D2H of the decision row (bytes summed over "
                        "ranks); the gradient of step i+1 is copied on a side stream into a second "
                        "device buffer while step i runs (serial_value: copy, step, read back in turn)")}

    ms_step = res["ms"] / args.steps
    one_launch = world > 1 and args.collective == "symm" and args.flag_exchange == "fused"
    # roofline of the update kernel: its per-launch time on local steps (at
    # N > 1 with the one-launch step this also holds the vote exchange)
    kms = sorted(modes["all_local"]["kernel_ms"])
    timed_on = "all_local mode, CUDA events around every launch on the launching stream"
    if not kms:  # --graph / --no-kernel-events: bound the kernel by the whole local step
        kms = [modes["all_local"]["ms"] / args.steps]
        timed_on = ("all_local step time under graph replay (upper bound of the kernel time)" if args.graph else
                    "all_local step time without per-launch events (upper bound of the kernel time)")
    k_mean = sum(kms) / len(kms)
    bytes_per_launch = (20 if args.momentum else 12) * P
    if args.no_fuse:
        bytes_per_launch = 4 * P
    order_eff = resolve_order(args.order, P, world)
    if one_launch and order_eff == "norm_first":
        bytes_per_launch += 4 * P  # norm pass first, then the plain update (both inside the launch)
    achieved = bytes_per_launch / (k_mean * 1e-3) / 1e9
    kernel_name = ("ss_update_norm_signal_f32 (K13+K2: fused SGD-momentum-wd update + ||g||^2 + signal step)"
                   if not args.no_fuse else "ss_norm_signal_f32 (K1+K2)")
    traffic_key = "sgd_kernel" if not args.no_fuse else "norm_kernel"
    if one_launch:
        kernel_name = ("ss_step_symm_f32 (one cooperative launch: K13+K2, the P2P vote exchange in the last "
                       "block, and on sync steps the NVLink mean by every block of the same grid; timed on "
                       "local steps)")
        traffic_key = "step_kernel_local"  # update-first local step; ncu runs single-GPU commands only
    sync_frac = sum(1 for d in res["decisions"] if d) / len(res["decisions"])
    line = {
        "metric": METRIC,
        "value": world * 1e3 / ms_step,
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic (seeded randn gradients resident in HBM; random-init flat parameters)",
        "config": workload_config(args, world),
        "observed_sync_frac": sync_frac,
        "roofline": {
            "bound": "hbm",
            "kernel": kernel_name,
            "achieved": achieved,
            "peak": hbm_peak,
            "peak_source": hbm_src,
            "unit": "GB/s",
            "frac": achieved / hbm_peak,
            "traffic": traffic_from_profiles(traffic_key, P),
            "traffic_source": traffic_from_profiles(traffic_key, P, field="source"),
            "algorithmic_bytes_per_launch": bytes_per_launch,
            "kernel_ms_mean": k_mean,
            "kernel_ms_median": kms[len(kms) // 2],
            "kernel_share_of_local_step": k_mean / (modes["all_local"]["ms"] / args.steps),
            "timed_on": timed_on,
        },
        "gpu_launches": res["launches"],
        "clocks": clocks.summary(),
        "modes": {},
    }
    if world == 1 and not args.no_fuse and res["launches"] == args.steps:
        # N = 1: the headline's timed region is exactly one K13 launch per step,
        # back to back without per-launch events (launches overlap their ramp
        # through programmatic dependent launch): bytes per launch / (region / launches)
        line["roofline"]["back_to_back"] = {
            "achieved": bytes_per_launch / (ms_step * 1e-3) / 1e9,
            "frac": bytes_per_launch / (ms_step * 1e-3) / 1e9 / hbm_peak,
            "ms_per_launch": ms_step,
            "timed_on": "the headline's timed region (CUDA events around it) / its K13 launches"}
    for name, m in modes.items():
        ent = {"steps_per_s": world * args.steps / (m["ms"] / 1e3), "ms_per_step": m["ms"] / args.steps,
               "kernel_ms_mean": sum(m["kernel_ms"]) / len(m["kernel_ms"]) if m["kernel_ms"] else None}
        ent.update(exchange_stats(m, P, world))
        ent["delta"] = 1e9 if name == "all_local" else 0.0
        if name == "all_sync" and one_launch and order_eff != "update_first":
            ent["note"] = ("delta = 0: every step is sync before ||g||^2 is known, so the one-launch step "
                           "takes the known-sync pass (no norm sweep, mean overlapped from the first tile)")
        line["modes"][name] = ent
    for case, (m, sched) in replays.items():
        line["modes"][f"replay_{case}"] = {
            "steps_per_s": world * args.steps / (m["ms"] / 1e3), "ms_per_step": m["ms"] / args.steps,
            "sync_frac": sum(1 for d in m["decisions"] if d) / max(1, len(m["decisions"])),
            "pattern": (f"post-warmup agreed decisions of the reference's golden {case} trace "
                        f"({len(sched)} steps, cycled): not periodic, unlike the headline mix"),
        }
    line.update({"exchange": exchange_stats(res, P, world)} if world > 1 else {})
    if one_launch and c2 is not None:
        line["exchange"] = c2
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_run(1, P, 3, 1, args, args.cpu_seconds)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "host_cpus", "cpu_model", "kind",
                                                    "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def model_bench(args, dev, comm, rank, world, local, hbm_peak, hbm_src):
    """BASELINE configs 1-3: steps/s of fwd/bwd (stock PyTorch) + the SelSync hot path."""
    import torch
    import torch.distributed as dist

    from paper_2307_07950_b200 import kernels as K
    from paper_2307_07950_b200 import workloads as W
    from paper_2307_07950_b200.train import SelSyncTrainer

    wl = W.build(args.workload, dev, rank=rank, world=world)
    P = W.parameter_count(wl.model)
    tr = SelSyncTrainer(wl, delta=args.delta, warmup=args.sel_warmup, group=comm,
                        collective=args.collective if world > 1 else None,
                        flag_exchange=(args.flag_exchange if args.collective == "symm" else "nccl"),
                        trace_capacity=1 << 14, profile=True)
    st = tr.step
    graph = args.graph
    if graph:
        st.profile = False
        batch0 = wl.make_batch(0)
        static = tuple(t.clone() for t in batch0)
        tr.capture(static, warmup_iters=max(3, args.warmup))

        def one_step():
            nb = wl.make_batch(tr.iteration)
            if nb[0].data_ptr() != static[0].data_ptr():
                for d_, s_ in zip(static, nb):
                    d_.copy_(s_, non_blocking=True)
            tr.replay_step()
    else:
        def one_step():
            tr.train_step()
        for _ in range(args.warmup):
            one_step()
    torch.cuda.synchronize()
    comm.barrier(dev)
    clocks = ClockSampler(local)
    l0, k0, d0 = K.LAUNCHES, len(st.kernel_events), st.steps_done
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    a.record()
    for _ in range(args.steps):
        one_step()
    b.record()
    torch.cuda.synchronize()
    clocks.stop()
    st.synchronize()
    comm.barrier(dev)
    ms = comm.max_float(a.elapsed_time(b), dev)
    launches = K.LAUNCHES - l0 if not graph else args.steps  # one SelSync kernel per replayed graph
    kms = st.kernel_ms()[k0:]
    dec = st.decisions()[d0 - st.steps_done:]
    # roofline of the update launch on local steps (sync steps add the mean)
    local_ms = [t for t, d in zip(kms, dec) if not d] if world > 1 else kms
    k_mean = sum(local_ms) / len(local_ms) if local_ms else None
    nbytes = (20 if wl.momentum else 12) * st.params.numel()
    achieved = nbytes / (k_mean * 1e-3) / 1e9 if k_mean else None
    # e2e: public blocking API, batch copied from pinned host memory, loss read back
    e2e = None
    if not args.no_e2e and not graph:
        hb = [t.cpu().pin_memory() for t in wl.make_batch(0)]
        db = [torch.empty_like(t, device=dev) for t in hb]
        lh = torch.empty(1, pin_memory=True)
        for i in range(args.warmup + args.steps):
            if i == args.warmup:
                torch.cuda.synchronize()
                comm.barrier(dev)
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record()
            for d_, h_ in zip(db, hb):
                d_.copy_(h_, non_blocking=True)
            loss, _ = tr.train_step(tuple(db), wait=True)
            lh.copy_(loss.reshape(1), non_blocking=True)
            torch.cuda.current_stream().synchronize()
        eb.record()
        torch.cuda.synchronize()
        ems = comm.max_float(ea.elapsed_time(eb), dev)
        e2e = {"value": world * args.steps / (ems / 1e3), "unit": "steps/s",
               "h2d_bytes_per_step": wl.host_batch_bytes * world, "d2h_bytes_per_step": 4 * world,
               "ms_per_step": ems / args.steps}
    line = {
        "metric": METRIC, "value": world * args.steps / (ms / 1e3), "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic tensors of the config's shape, random-init weights",
        "config": {"workload": f"{args.workload} (BASELINE configs): stock PyTorch fwd/bwd + SelSync hot path"
                               + (", fwd + bwd + step captured in one CUDA graph" if graph else ""),
                   "P": P, "P_padded": st.params.numel(), "delta": args.delta, "warmup": args.sel_warmup,
                   "momentum": wl.momentum, "weight_decay": wl.weight_decay, "n_workers": world,
                   "parallelism": f"dp{world} (SelSync replicas)",
                   "value_counts": "worker-steps: N ranks x K steps / (max-over-ranks device time)"},
        "observed_sync_frac": sum(dec) / max(1, len(dec)),
        "roofline": {"bound": "hbm", "kernel": "SelSync update launch (K13+K2[+exchange])",
                     "achieved": achieved, "peak": hbm_peak, "peak_source": hbm_src,
                     "unit": "GB/s", "frac": achieved / hbm_peak if achieved else None, "traffic": None,
                     "kernel_ms_mean": k_mean,
                     "timed_on": ("not timed inside a CUDA graph (run without --graph)" if graph else
                                  "local steps" if world > 1 else "all steps"),
                     "hot_path_share_of_step": sum(kms) / len(kms) / (ms / args.steps) if kms else None},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def replay_schedules():
    """Gradient-ring schedules that reproduce the agreed decisions of the
    reference's golden n4_mixed / n8_mixed runs (tests/golden, made by the
    unmodified reference): with smoothing 1 and delta 0.3 a step syncs iff its
    gradient scale differs from the previous step's (ring 0 = 1.0, ring 2 = 1.5)."""
    import numpy as np

    z = np.load(ROOT / "tests" / "golden" / "selsync_cases.npz")
    meta = json.loads(bytes(z["meta_json"]).decode())
    out = {}
    for case in ("n4_mixed", "n8_mixed"):
        dec = z[f"{case}/decision"][:, 0][int(meta[case]["warmup"]):]
        sched, cur = [], 0
        for d in dec:
            if d:
                cur = 2 - cur
            sched.append(cur)
        if sched[0] == sched[-1]:  # the cycle's wrap-around must be local: same buffer
            out[case] = sched
        else:
            out[case] = sched + sched  # even number of switches over the doubled cycle
    return out


def exchange_stats(m, P, world):
    """C1+C2 timing per step kind. Symmetric path: one event pair per step
    (local steps = flag agreement + early exit); NCCL path: pairs on sync
    steps only. busbw = (4P / t) * 2(N-1)/N (nccl-tests convention)."""
    if world < 2 or not m["sync_ms"]:
        return {}
    sms, dec = m["sync_ms"], m["decisions"]
    if len(sms) == len(dec):
        on_sync = [t for t, d in zip(sms, dec) if d]
        on_local = [t for t, d in zip(sms, dec) if not d]
    else:
        on_sync, on_local = sms, []
    out = {}
    if on_local:
        out["local_exchange_us_mean"] = 1e3 * sum(on_local) / len(on_local)
    if on_sync:
        t = sum(on_sync) / len(on_sync)
        algbw = 4 * P / (t * 1e-3) / 1e9
        busbw = algbw * 2 * (world - 1) / world
        out["sync_exchange_ms_mean"] = t
        out["nvlink"] = {"busbw": busbw, "algbw": algbw, "unit": "GB/s",
                         "peak_nominal": NVLINK_NOMINAL_GBS, "frac_nominal": busbw / NVLINK_NOMINAL_GBS,
                         "ref_nccl_allreduce_busbw_1GiB_8gpu": NVLINK_ALLREDUCE_MEASURED_GBS,
                         "frac_of_ref": busbw / NVLINK_ALLREDUCE_MEASURED_GBS}
    return out


def traffic_from_profiles(kernel, P, field="dram_bytes_per_launch"):
    """dram read+write bytes per launch of THIS roofline kernel (sgd_kernel =
    K13; step_kernel_local = the one-launch step kernel's update-first local
    step, captured through a world-1 group because ncu only profiles
    single-GPU commands) from the committed ncu --set full summaries at the
    same P, if one exists; field="source" names the capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        ent = json.loads(p.read_text()).get(kernel, {}).get(str(P))
        return None if ent is None else ent[field]
    except Exception:
        return None


if __name__ == "__main__":
    main()
