"""Decision-trace output in the reference's metrics schema (SURVEY §8 f, row 3).

``SelSyncStep.records()`` / ``ReplicaSelSync.records()`` read the device trace
ring in batches; this module writes them as ``metrics.jsonl`` rows with the
exact field set of the reference's ``MetricsRecord`` (metrics.py:23-48) and
reads them back, so the reference's own tooling (``selsync replay-trace``,
LSSR summaries) works on B200 runs, and ``replay_trace`` re-implements the
counterfactual delta grid of cli.py:53-72 on the same rows.

Columns the reference fills from its parameter-server byte ledger are filled
with what this path actually moves per rank: the 4-byte flag word every step
and, on sync steps, the 4P-byte parameter payload (in and out).
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path
from typing import Iterable, Optional

from .errors import ConfigError
from .signal import DeltaThreshold, replay_decisions

FIELDS = ("step", "worker_id", "loss", "grad_norm_sq", "ewma", "delta_g", "decision", "bytes_sent",
          "bytes_received", "step_duration", "lr")


def to_metrics_rows(records: Iterable[dict], n_params: int, losses: Optional[dict] = None,
                    durations: Optional[dict] = None) -> list[dict]:
    """Map device trace records onto MetricsRecord rows (metrics.py:23-48)."""
    rows = []
    for r in records:
        sync = r["decision"] == "sync"
        payload = 4 + (4 * n_params if sync else 0)
        loss = (losses or {}).get(r["step"], math.nan)
        rows.append({
            "step": int(r["step"]),
            "worker_id": int(r["worker_id"]),
            "loss": float(loss),
            "grad_norm_sq": float(r["grad_norm_sq"]),
            "ewma": float(r["ewma"]),
            "delta_g": None if r["delta_g"] is None else float(r["delta_g"]),
            "decision": "sync" if sync else "local",
            "bytes_sent": payload,
            "bytes_received": payload,
            "step_duration": float((durations or {}).get(r["step"], 0.0)),
            "lr": float(r.get("lr", 0.0)),
        })
    return rows


def write_metrics_jsonl(rows: Iterable[dict], path) -> None:
    """One JSON object per line, keys sorted, rows ordered by (step, worker_id)
    -- the reference's format (metrics.py:129-133)."""
    with open(path, "w", encoding="utf-8") as fh:
        for row in sorted(rows, key=lambda r: (r["step"], r["worker_id"])):
            fh.write(json.dumps({k: row[k] for k in FIELDS}, sort_keys=True) + "\n")


def load_metrics_jsonl(path) -> list[dict]:
    rows = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            if not line.strip():
                continue
            try:
                d = json.loads(line)
            except json.JSONDecodeError as exc:
                raise ConfigError(f"{path}:{lineno}: {exc}") from exc
            missing = [k for k in FIELDS if k not in d]
            if missing:
                raise ConfigError(f"{path}:{lineno}: missing fields {missing}")
            if d["decision"] not in ("sync", "local"):
                raise ConfigError(f"{path}:{lineno}: bad decision {d['decision']!r}")
            rows.append({k: d[k] for k in FIELDS})
    return rows


def lssr(rows: list[dict], worker: int = 0) -> float:
    """Local-to-sync step ratio: fraction of purely local steps (metrics.py:71-79)."""
    mine = [r for r in rows if r["worker_id"] == worker]
    if not mine:
        raise ConfigError(f"trace has no records for worker {worker}")
    return sum(1 for r in mine if r["decision"] == "local") / len(mine)


def replay_trace(rows: list[dict], worker: int, deltas: list[float], warmup: int) -> list[tuple[float, int]]:
    """Counterfactual sync counts per delta for one worker's recorded Delta trace (cli.py:53-72)."""
    trace = [r["delta_g"] for r in sorted(rows, key=lambda r: r["step"]) if r["worker_id"] == worker]
    if not trace:
        raise ConfigError(f"trace has no records for worker {worker}")
    grid = sorted(float(d) for d in deltas)
    for d in grid:
        DeltaThreshold(d)
    return [(d, replay_decisions(trace, warmup, d)) for d in grid]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="counterfactual delta replay of a B200 SelSync trace")
    ap.add_argument("--trace", required=True)
    ap.add_argument("--deltas", required=True)
    ap.add_argument("--worker", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=25)
    a = ap.parse_args(argv)
    counts = replay_trace(load_metrics_jsonl(a.trace), a.worker,
                          [float(x) for x in a.deltas.split(",")], a.warmup)
    for d, c in counts:
        print(f"delta={d:g} syncs={c}")
    for (d1, c1), (d2, c2) in zip(counts, counts[1:]):
        if c2 > c1:
            print(f"monotonicity violated: delta={d2:g} syncs={c2} > delta={d1:g} syncs={c1}", file=sys.stderr)
            return 1
    print("monotone: sync counts nonincreasing in delta")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
