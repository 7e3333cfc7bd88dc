"""Golden learning-rate schedule vectors from the UNMODIFIED reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_lr_golden.py

Evaluates ``selsync.model.lr_at`` (model.py:252-258) and the worker's
``lr_for`` mapping step -> epoch = step // steps_per_epoch
(strategies.py:155-156) for a grid of ``LrSchedule`` objects (per_step and
per_epoch milestones, recurring decays, boundaries at 0, factors > 1), and
records which constructor arguments the reference rejects (model.py:237-249).
Writes tests/golden/lr_cases.json (the reference is not present on GPU boxes).
"""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from selsync.errors import ConfigError  # noqa: E402
from selsync.model import LrSchedule, lr_at  # noqa: E402

SCHEDULES = [
    dict(initial_lr=0.5, milestones=[], mode="per_step"),
    dict(initial_lr=0.1, milestones=[[110, 0.1]], mode="per_epoch"),
    dict(initial_lr=2.0, milestones=[[2000, 0.8], [4000, 0.8]], mode="per_step"),
    dict(initial_lr=0.1, milestones=[[0, 0.5], [3, 0.1], [7, 0.1]], mode="per_step"),
    dict(initial_lr=0.1, milestones=[[0, 0.5], [3, 0.1], [7, 0.1]], mode="per_epoch"),
    dict(initial_lr=0.05, milestones=[[1, 2.0], [2, 3.0], [5, 0.25]], mode="per_epoch"),
    dict(initial_lr=0.3, milestones=[[k * 100, 0.9] for k in range(1, 20)], mode="per_step"),
    dict(initial_lr=1e-3, milestones=[[150, 0.1], [225, 0.1]], mode="per_epoch"),
]
POSITIONS = [0, 1, 2, 3, 4, 6, 7, 8, 99, 100, 109, 110, 111, 149, 150, 224, 225, 1999, 2000, 3999, 4000,
             10_000]
STEPS_PER_EPOCH = [1, 7, 390]
BAD = [dict(initial_lr=0.0), dict(initial_lr=-1.0), dict(initial_lr=0.1, milestones=[[5, 0.1], [5, 0.1]]),
       dict(initial_lr=0.1, milestones=[[6, 0.1], [5, 0.1]]), dict(initial_lr=0.1, milestones=[[5, -1.0]]),
       dict(initial_lr=0.1, milestones=[[5, 0.0]]), dict(initial_lr=0.1, mode="per_batch")]


def make(d):
    return LrSchedule(d["initial_lr"], tuple(tuple(m) for m in d.get("milestones", [])), d.get("mode", "per_step"))


def main():
    cases = []
    for d in SCHEDULES:
        s = make(d)
        rows = []
        for step in POSITIONS:
            for spe in STEPS_PER_EPOCH:
                epoch = step // spe  # WorkerContext.lr_for, strategies.py:155-156
                rows.append([step, epoch, lr_at(s, step, epoch)])
        cases.append(dict(schedule=d, rows=rows))
    rejected = []
    for d in BAD:
        try:
            make(d)
            rejected.append(False)
        except ConfigError:
            rejected.append(True)
    out = dict(cases=cases, bad=BAD, rejected=rejected)
    (HERE / "lr_cases.json").write_text(json.dumps(out, indent=0, sort_keys=True) + "\n")
    print("wrote", HERE / "lr_cases.json", sum(len(c["rows"]) for c in cases), "rows")


if __name__ == "__main__":
    main()
