"""Generate golden fixtures by running the UNMODIFIED reference.

Run in the build container (the reference is not present on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``selsync`` from /root/reference/pkg/src and drives the stock
``run_simulation`` (runtime.py:462-581) with the same ParameterServer /
WorkerContext wiring as the reference's own ``build`` fixture
(test_runtime.py:42-94). The only substitution is the gradient source:
``selsync.strategies.forward_backward`` is replaced by the seeded fp32
synthetic gradient of ``oracle.selsync_oracle.synthetic_grad32`` keyed by
(worker, step), which a tag sampler encodes into ``Batch.features``
(the sampler is duck-typed, strategies.py:143). Everything downstream of the
gradient -- ``grad @ grad``, observe/relative_change/decide, sgd_step, the
flag OR, the PS mean -- is the reference's own code.

Outputs ``tests/golden/selsync_cases.npz`` (traces, init and final params, a
few trajectory snapshots) and ``tests/golden/seldp_cases.npz`` (SelDP plans
and sampler index streams, data.py:178-419).
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))

import selsync.strategies as ref_strategies  # noqa: E402
from selsync.data import (  # noqa: E402
    ChunkSampler,
    Dataset,
    bind_plan,
    plan_defdp,
    plan_seldp,
    split_chunks,
)
from selsync.model import Batch, LrSchedule, ModelSpec  # noqa: E402
from selsync.runtime import ClusterConfig, ParameterServer, SimTransport, run_simulation  # noqa: E402
from selsync.strategies import LogicalCosts, SelSyncConfig, WorkerContext  # noqa: E402

from oracle.selsync_oracle import synthetic_grad32  # noqa: E402

GRAD_SEED = 1234


class TagSampler:
    """Batch.features = [[worker, step]] so the patched forward_backward can
    key its synthetic gradient; labels are unused."""

    def __init__(self, worker: int):
        self.worker = worker
        self.step = 0

    def next_batch(self) -> Batch:
        b = Batch(np.array([[float(self.worker), float(self.step)]]), np.zeros(1, dtype=np.int64))
        self.step += 1
        return b


def synthetic_forward_backward(params, batch, spec):
    worker, step = (int(v) for v in batch.features[0])
    g = synthetic_grad32(GRAD_SEED, worker, step, params.values.size).astype(np.float64)
    return 0.0, g


def run_case(n, d, steps, delta, warmup, smoothing, lr, aggregation, init_seed, name_for_metrics=None):
    ref_strategies.forward_backward = synthetic_forward_backward
    spec = ModelSpec(input_dim=d, hidden_dims=(), num_classes=2, init_seed=init_seed)
    strategy = SelSyncConfig(delta=delta, aggregation=aggregation, warmup=warmup, smoothing=smoothing)
    sched = LrSchedule(initial_lr=lr)
    ps = ParameterServer(spec, strategy, n, sched, steps_per_epoch=10**6)
    cluster = ClusterConfig(n_workers=n, transport=SimTransport(schedule_seed=0))
    ctxs = [
        WorkerContext(
            worker_id=w, n_workers=n, spec=spec, sampler=TagSampler(w), strategy=strategy,
            schedule=sched, steps_per_epoch=10**6, budget_steps=steps, eval_every=10**9,
            logical_costs=LogicalCosts(), capture=lambda s: True,
        )
        for w in range(n)
    ]
    res = run_simulation(ps, ctxs, cluster)
    if name_for_metrics is not None:
        from selsync.metrics import write_metrics_jsonl
        from selsync.signal import replay_decisions

        write_metrics_jsonl(res.rows, HERE / f"{name_for_metrics}_metrics.jsonl")
        trace = [r.delta_g for r in sorted(res.rows, key=lambda r: r.step) if r.worker_id == 0]
        grid = [0.0, 0.005, 0.01, 0.02, 0.05, 0.1, 1.0]
        (HERE / f"{name_for_metrics}_replay.json").write_text(json.dumps(
            {"worker": 0, "warmup": warmup, "grid": grid,
             "syncs": [replay_decisions(trace, warmup, dd) for dd in grid]}))
    P = 2 * d + 2
    gn = np.zeros((steps, n))
    ew = np.zeros((steps, n))
    dg = np.full((steps, n), np.nan)
    dec = np.zeros((steps, n), dtype=bool)
    for r in res.rows:
        gn[r.step, r.worker_id] = r.grad_norm_sq
        ew[r.step, r.worker_id] = r.ewma
        if r.delta_g is not None:
            dg[r.step, r.worker_id] = r.delta_g
        dec[r.step, r.worker_id] = r.decision == "sync"
    traj = np.zeros((steps, n, P))
    for w in range(n):
        for s, vals in res.worker_reports[w]["trajectory"]:
            traj[s, w] = vals
    finals = np.stack([res.finals[w] for w in range(n)])
    return dict(init=res.init_values, grad_norm_sq=gn, ewma=ew, delta_g=dg, decision=dec,
                finals=finals, trajectory=traj)


# name: (N, d, steps, delta, warmup, smoothing, lr, aggregation, init_seed)
CASES = {
    # BASELINE configs[0]: 2 workers, delta 0.3, EWMA window 25, P = 1002 (degenerate: warmup only)
    "cfg0_n2_d0.3": (2, 500, 60, 0.3, 25, None, 0.05, "params", 3),
    "n1_mixed": (1, 300, 50, 0.003, 3, None, 0.1, "params", 1),
    "n2_lam0.5": (2, 257, 50, 0.05, 3, 0.5, 0.1, "params", 2),
    "n4_mixed": (4, 500, 60, 0.02, 5, None, 0.1, "params", 3),
    "n8_mixed": (8, 200, 60, 0.05, 25, None, 0.05, "params", 4),
    "n4_delta0": (4, 100, 30, 0.0, 1, None, 0.1, "params", 5),
    "n4_huge": (4, 100, 40, 1e9, 5, None, 0.1, "params", 6),
    "n4_grads": (4, 300, 50, 0.02, 5, None, 0.1, "grads", 7),
    "n2_grads": (2, 301, 50, 0.05, 3, 0.5, 0.1, "grads", 8),
}


def seldp_fixture():
    """SelDP planner + ChunkSampler index streams (data.py:178-419)."""
    out = {}
    n_samples = 1000
    feats = np.arange(n_samples, dtype=np.float64)[:, None]
    ds = Dataset(feats, np.zeros(n_samples, dtype=np.int64) % 2, num_classes=2)
    for n in (1, 2, 3, 4, 8):
        split = split_chunks(n_samples, n, seed=5)
        out[f"perm_n{n}"] = split.permutation
        out[f"bounds_n{n}"] = np.array(split.bounds, dtype=np.int64)
        for scheme, planner in (("seldp", plan_seldp), ("defdp", plan_defdp)):
            for w in range(n):
                plan = bind_plan(planner(w, n), split)
                out[f"{scheme}_order_n{n}_w{w}"] = np.array(plan.chunk_order, dtype=np.int64)
                sampler = ChunkSampler(ds, split, plan, batch_size=16, seed=100)
                idx, src = [], []
                for _ in range(3 * (sampler.epoch_length // 16) + 2):
                    b = sampler.next_batch()
                    idx.append(b.features[:, 0].astype(np.int64))
                    src.append(b.source_chunk)
                out[f"{scheme}_batches_n{n}_w{w}"] = np.stack(idx)
                out[f"{scheme}_sources_n{n}_w{w}"] = np.array(src, dtype=np.int64)
    return out


def main():
    arrays = {}
    meta = {}
    for name, args in CASES.items():
        res = run_case(*args, name_for_metrics=name if name == "n4_mixed" else None)
        n, d, steps, delta, warmup, smoothing, lr, agg, init_seed = args
        meta[name] = dict(n=n, d=d, P=2 * d + 2, steps=steps, delta=delta, warmup=warmup,
                          smoothing=smoothing, lr=lr, aggregation=agg, init_seed=init_seed,
                          grad_seed=GRAD_SEED,
                          syncs=int(res["decision"][:, 0].sum()))
        snaps = sorted({0, warmup, steps // 2, steps - 1})
        arrays[f"{name}/init"] = res["init"]
        for k in ("grad_norm_sq", "ewma", "delta_g", "decision", "finals"):
            arrays[f"{name}/{k}"] = res[k]
        arrays[f"{name}/snap_steps"] = np.array(snaps)
        arrays[f"{name}/snaps"] = res["trajectory"][snaps]
        print(name, meta[name])
    arrays["meta_json"] = np.frombuffer(json.dumps(meta, sort_keys=True).encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "selsync_cases.npz", **arrays)
    np.savez_compressed(HERE / "seldp_cases.npz", **seldp_fixture())


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    main()
