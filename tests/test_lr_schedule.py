"""lr_at / LrSchedule (model.py:224-258) against vectors produced by the
unmodified reference (tests/golden/make_lr_golden.py): per_step and per_epoch
milestones, the worker's step -> epoch mapping (strategies.py:155-156) and the
reference's constructor validation; plus the reference's own known answers
(test_model.py:222-245)."""

import json
from pathlib import Path

import pytest

from oracle import selsync_oracle as O
from paper_2307_07950_b200 import ConfigError
from paper_2307_07950_b200.model import LrSchedule, lr_at

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "lr_cases.json").read_text())


def make(cls, d):
    return cls(d["initial_lr"], tuple(tuple(m) for m in d.get("milestones", [])), d.get("mode", "per_step"))


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_lr_at_matches_reference_vectors(i):
    case = GOLD["cases"][i]
    ours, oracle = make(LrSchedule, case["schedule"]), make(O.LrSchedule, case["schedule"])
    for step, epoch, want in case["rows"]:
        assert lr_at(ours, step, epoch) == want  # same float operations, bit-exact
        assert O.lr_at(oracle, step, epoch) == want


def test_lr_schedule_validation_matches_reference():
    for d, rejected in zip(GOLD["bad"], GOLD["rejected"]):
        assert rejected
        with pytest.raises(ConfigError):
            make(LrSchedule, d)


def test_reference_known_answers():
    assert lr_at(LrSchedule(0.5), 10_000, 99) == 0.5
    s = LrSchedule(0.1, ((110, 0.1),), mode="per_epoch")
    assert lr_at(s, 0, 120) == pytest.approx(0.01)
    assert lr_at(s, 0, 109) == pytest.approx(0.1)
    assert lr_at(s, 0, 110) == pytest.approx(0.01)
    s = LrSchedule(2.0, ((2000, 0.8), (4000, 0.8)), mode="per_step")
    assert lr_at(s, 4000, 0) == pytest.approx(1.28)
    assert lr_at(s, 3999, 0) == pytest.approx(1.6)
