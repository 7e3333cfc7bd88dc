"""SelSyncConfig validation (strategies.py:106-121) and flag-word semantics
(wire.py:126-155, test_runtime.py:178-191)."""

import pytest

from paper_2307_07950_b200 import (
    ConfigError,
    SelSyncConfig,
    SignalError,
    any_flag,
    flag_word,
    flag_word_size,
    flags_in_word,
    or_words,
)
from paper_2307_07950_b200.errors import ProtocolError
from paper_2307_07950_b200.wire import votes_to_word


def test_config_defaults_and_validation():
    c = SelSyncConfig(delta=0.3)
    assert (c.aggregation, c.warmup, c.smoothing) == ("params", 25, None)
    assert c.smoothing_for(8) == pytest.approx(0.08)
    assert SelSyncConfig(delta=0.3, smoothing=0.5).smoothing_for(8) == 0.5
    with pytest.raises(ConfigError):
        SelSyncConfig(delta=0.3, aggregation="bogus")
    with pytest.raises(SignalError):
        SelSyncConfig(delta=-1.0)
    with pytest.raises(ConfigError):
        SelSyncConfig(delta=0.3, warmup=0)
    with pytest.raises(ConfigError):
        SelSyncConfig(delta=0.3, smoothing=1.5)
    with pytest.raises(ConfigError):
        SelSyncConfig(delta=0.3, nesterov=True)
    with pytest.raises(ConfigError):
        SelSyncConfig(delta=0.3, momentum=-0.1)


def test_config_json_round_trip():
    ref_obj = {"kind": "selsync", "delta": 0.5, "aggregation": "grads", "warmup": 10, "smoothing": None}
    c = SelSyncConfig.from_json(ref_obj)
    assert c == SelSyncConfig(delta=0.5, aggregation="grads", warmup=10)
    assert SelSyncConfig.from_json(c.to_json()) == c
    with pytest.raises(ConfigError):
        SelSyncConfig.from_json({"kind": "bsp"})


def test_flag_words():
    assert flag_word(10, {0, 9}) == b"\x01\x02"
    assert flag_word(8, set()) == b"\x00"
    assert [flag_word_size(n) for n in (8, 9, 16, 17)] == [1, 2, 2, 3]
    merged = or_words([flag_word(12, {w}) for w in (1, 4, 11)], 12)
    assert any_flag(merged)
    assert [i for i, b in enumerate(flags_in_word(merged, 12)) if b] == [1, 4, 11]
    assert not any_flag(flag_word(12, set()))
    assert votes_to_word([0, 1, 0, 1]) == b"\x0a"
    with pytest.raises(ProtocolError):
        flag_word(4, {4})


def test_int_max_equals_bit_or():
    # the device exchange is allreduce-MAX over 0/1 words: identical to the OR
    import itertools

    for votes in itertools.product([0, 1], repeat=5):
        assert (max(votes) == 1) == any_flag(votes_to_word(votes))


def test_integration_doc_names_resolve():
    """Every name INTEGRATION.md imports from the package resolves (lazily)."""
    import paper_2307_07950_b200 as S

    for name in ("observe", "decide", "DeltaThreshold", "GradSignalState", "default_smoothing",
                 "SelSyncConfig", "split_chunks", "plan_seldp", "bind_plan", "ChunkSampler",
                 "FlatParameters", "SelSyncStep", "LrSchedule", "lr_at", "SelSyncTrainer",
                 "TensorListSelSyncStep", "ReplicaSelSync", "RankGroup"):
        assert getattr(S, name) is not None, name


def test_auto_order_picks_update_first_for_small_models():
    """order="auto" (the SelSyncStep default): the overlapped norm-first pass
    only where it was measured faster on sync steps (profiles/r02_order_size)."""
    from paper_2307_07950_b200.collectives import resolve_order

    assert resolve_order("auto", 16_000_000, 2) == "update_first"
    assert resolve_order("auto", 32_000_000, 2) == "adaptive"
    assert resolve_order("auto", 4_000_000, 4) == "update_first"
    assert resolve_order("auto", 16_000_000, 4) == "adaptive"
    assert resolve_order("auto", 100_000_000, 8) == "adaptive"
    for o in ("update_first", "norm_first", "adaptive", "nan_safe"):
        assert resolve_order(o, 1000, 2) == o
