"""Trace output in the reference's metrics.jsonl schema (metrics.py:23-48,
:129-141) and the counterfactual replay of cli.py:53-72, pinned against a
file and replay counts the unmodified reference produced
(tests/golden/make_golden.py, case n4_mixed)."""

import json
from pathlib import Path

import pytest

from paper_2307_07950_b200 import trace as T
from paper_2307_07950_b200.errors import ConfigError

GOLD = Path(__file__).resolve().parent / "golden"


def test_reference_file_round_trips_byte_identical(tmp_path):
    rows = T.load_metrics_jsonl(GOLD / "n4_mixed_metrics.jsonl")
    assert len(rows) == 60 * 4
    out = tmp_path / "metrics.jsonl"
    T.write_metrics_jsonl(rows, out)
    assert out.read_bytes() == (GOLD / "n4_mixed_metrics.jsonl").read_bytes()


def test_replay_counts_match_reference(capsys):
    want = json.loads((GOLD / "n4_mixed_replay.json").read_text())
    rows = T.load_metrics_jsonl(GOLD / "n4_mixed_metrics.jsonl")
    got = T.replay_trace(rows, want["worker"], want["grid"], want["warmup"])
    assert [c for _, c in got] == want["syncs"]
    rc = T.main(["--trace", str(GOLD / "n4_mixed_metrics.jsonl"), "--deltas",
                 ",".join(map(str, want["grid"])), "--worker", "0", "--warmup", str(want["warmup"])])
    assert rc == 0 and "monotone" in capsys.readouterr().out


def test_to_metrics_rows_and_lssr():
    recs = [dict(step=s, worker_id=0, grad_norm_sq=1.0 + s, ewma=1.0, delta_g=None if s == 0 else 0.1,
                 decision="sync" if s % 3 == 0 else "local", lr=0.1) for s in range(9)]
    rows = T.to_metrics_rows(recs, n_params=100)
    assert rows[0]["bytes_sent"] == 4 + 400 and rows[1]["bytes_sent"] == 4
    assert set(rows[0]) == set(T.FIELDS)
    assert T.lssr(rows) == pytest.approx(6 / 9)


def test_loader_rejects_malformed(tmp_path):
    p = tmp_path / "bad.jsonl"
    p.write_text('{"step": 0}\n')
    with pytest.raises(ConfigError):
        T.load_metrics_jsonl(p)
