"""SelDP partitioner + samplers: index-exact against the reference's own
streams (tests/golden/seldp_cases.npz, produced by make_golden.py from
data.py:178-419), plus the reference's structural properties."""

import numpy as np
import pytest

from paper_2307_07950_b200 import (
    ChunkSampler,
    ConfigError,
    TokenStreamSampler,
    bind_plan,
    plan_call_count,
    plan_defdp,
    plan_seldp,
    split_chunks,
)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_split_matches_reference(n, seldp_golden):
    split = split_chunks(1000, n, seed=5)
    np.testing.assert_array_equal(split.permutation, seldp_golden[f"perm_n{n}"])
    np.testing.assert_array_equal(np.array(split.bounds), seldp_golden[f"bounds_n{n}"])


@pytest.mark.parametrize("scheme,planner", [("seldp", plan_seldp), ("defdp", plan_defdp)])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_sampler_streams_match_reference(scheme, planner, n, seldp_golden):
    split = split_chunks(1000, n, seed=5)
    for w in range(n):
        plan = bind_plan(planner(w, n), split)
        np.testing.assert_array_equal(plan.chunk_order, seldp_golden[f"{scheme}_order_n{n}_w{w}"])
        sampler = ChunkSampler(1000, split, plan, batch_size=16, seed=100)
        want = seldp_golden[f"{scheme}_batches_n{n}_w{w}"]
        src = seldp_golden[f"{scheme}_sources_n{n}_w{w}"]
        for i in range(want.shape[0]):
            idx, s = sampler.next_indices()
            np.testing.assert_array_equal(idx, want[i])
            assert s == src[i]


def test_seldp_rotation_covers_every_chunk_once():
    for n in (2, 5, 8):
        orders = [plan_seldp(w, n).chunk_order for w in range(n)]
        for w, o in enumerate(orders):
            assert sorted(o) == list(range(n)) and o[0] == w
        # at every position k the N workers visit N distinct chunks
        for k in range(n):
            assert sorted(o[k] for o in orders) == list(range(n))


def test_dataset_gather_and_validation():
    feats = np.arange(40, dtype=np.float64)[:, None] * 2
    labels = np.arange(40) % 3
    split = split_chunks(40, 2, seed=1)
    s = ChunkSampler((feats, labels), split, bind_plan(plan_seldp(1, 2), split), 8, seed=3)
    f, y, src = s.next_batch()
    assert f.shape == (8, 1) and (y == (f[:, 0] / 2).astype(int) % 3).all() and src == 1
    with pytest.raises(ConfigError):
        split_chunks(3, 4, 0)
    with pytest.raises(ConfigError):
        plan_seldp(3, 3)
    with pytest.raises(ConfigError):
        ChunkSampler(40, split, bind_plan(plan_defdp(0, 2), split), 100, seed=0)


def test_planning_is_counted_once():
    before = plan_call_count()
    split = split_chunks(100, 4, seed=0)
    plans = [bind_plan(plan_seldp(w, 4), split) for w in range(4)]
    samplers = [ChunkSampler(100, split, p, 5, seed=1) for p in plans]
    for _ in range(50):
        for s in samplers:
            s.next_indices()
    assert plan_call_count() - before == 5  # no re-planning mid-run (data.py:24-34)


def test_token_stream_windows():
    n_tokens, bptt = 10_001, 35
    samplers = [TokenStreamSampler(n_tokens, bptt, w, 4, batch_size=8, seed=9) for w in range(4)]
    seen = set()
    for s in samplers:
        starts, src = s.next_windows()
        assert (starts % bptt == 0).all() and (starts + bptt + 1 <= n_tokens).all()
        seen.add(src)
    assert seen == {0, 1, 2, 3}  # SelDP: each worker starts on its own chunk
