"""Pin the CPU oracle before trusting it.

1. Known-answer tests restated from the reference's own suite
   (test_signal.py:28-182, test_model.py:162-183, test_strategies.py:193-217,
   test_runtime.py:178-191).
2. Bit-exact agreement of the oracle's N-worker restatement with the golden
   traces that the UNMODIFIED reference run_simulation produced
   (tests/golden/make_golden.py).
"""

import math

import numpy as np
import pytest

from conftest import case_names
from oracle import selsync_oracle as O


def observe_all(st, xs):
    for x in xs:
        st = O.observe(st, x)
    return st


class TestKnownAnswers:
    def test_smoothing(self):  # test_signal.py:29-39
        assert O.default_smoothing(16) == pytest.approx(0.16)
        assert O.default_smoothing(200) == 1.0
        assert O.default_smoothing(2) == pytest.approx(0.02)
        assert O.default_smoothing(1) == 0.05
        with pytest.raises(O.OracleConfigError):
            O.default_smoothing(0)

    def test_seed_and_blend(self):  # test_signal.py:47-57
        s = O.observe(O.SignalState(smoothing=0.5), 4.0)
        assert (s.ewma_current, s.ewma_previous, s.step_count) == (4.0, 0.0, 1)
        s = observe_all(O.SignalState(smoothing=0.5), [4.0, 2.0])
        assert s.ewma_current == pytest.approx(3.0)
        assert O.relative_change(s) == pytest.approx(0.25)

    def test_fixed_point_and_zero_cases(self):  # test_signal.py:59-62, 95-101
        s = observe_all(O.SignalState(smoothing=0.3), [7.5] * 40)
        assert O.relative_change(s) == 0.0
        assert O.relative_change(observe_all(O.SignalState(smoothing=0.5), [0.0, 0.0])) == 0.0
        assert O.relative_change(observe_all(O.SignalState(smoothing=0.5), [0.0, 2.0])) == math.inf

    def test_nan_negative(self):  # test_signal.py:72-80
        s = O.observe(O.SignalState(smoothing=0.5), 4.0)
        with pytest.raises(O.OracleSignalError):
            O.observe(s, float("nan"))
        with pytest.raises(O.OracleSignalError):
            O.observe(s, -1.0)

    def test_inclusive_threshold(self):  # test_signal.py:135-141
        s = observe_all(O.SignalState(smoothing=1.0, warmup=1), [1.0, 1.3])
        assert O.decide(s, 0.3) == "sync"
        assert O.decide(s, 0.30001) == "local"

    def test_warmup_forces_sync(self):  # test_signal.py:113-118
        s = O.SignalState(smoothing=0.5, warmup=5)
        for _ in range(5):
            s = O.observe(s, 1.0)
            assert O.decide(s, 1e9) == "sync"
        s = O.observe(s, 1.0)
        assert O.decide(s, 1e9) == "local"

    def test_sgd_and_mean(self):  # test_model.py:163-176, test_strategies.py:194-203
        w = np.ones(6)
        assert np.allclose(O.sgd_step(w, np.full(6, 0.5), 0.1), 0.95)
        assert np.array_equal(O.sgd_step(w, np.ones(6), 0.0), w)
        m = O.aggregate_mean([np.array([1.0, 3.0]), np.array([3.0, 1.0])])
        assert np.array_equal(m, [2.0, 2.0])

    def test_momentum_reduces_to_sgd(self):
        rng = np.random.default_rng(0)
        w, g = rng.standard_normal(9), rng.standard_normal(9)
        got, _ = O.sgd_momentum_step(w, g, None, 0.1, first=True)
        assert np.array_equal(got, O.sgd_step(w, g, 0.1))

    def test_momentum_matches_torch_sgd(self):
        torch = pytest.importorskip("torch")
        rng = np.random.default_rng(1)
        w0 = rng.standard_normal(17)
        p = torch.nn.Parameter(torch.tensor(w0, dtype=torch.float64))
        opt = torch.optim.SGD([p], lr=0.05, momentum=0.9, weight_decay=4e-4, nesterov=True)
        w, buf = w0.copy(), None
        for k in range(5):
            g = rng.standard_normal(17)
            p.grad = torch.tensor(g, dtype=torch.float64)
            opt.step()
            w, buf = O.sgd_momentum_step(w, g, buf, 0.05, 0.9, 0.0, 4e-4, True, first=(k == 0))
        np.testing.assert_allclose(p.detach().numpy(), w, rtol=1e-14, atol=1e-15)

    def test_flag_words(self):  # test_runtime.py:178-191
        assert O.flag_word(10, {0, 9}) == b"\x01\x02"
        assert O.flag_word(8, set()) == b"\x00"
        merged = O.or_words([O.flag_word(12, {w}) for w in (1, 4, 11)], 12)
        assert O.any_flag(merged)
        assert not O.any_flag(O.flag_word(12, set()))

    def test_replay_monotone(self):  # test_signal.py:168-182
        rng = np.random.default_rng(5)
        trace = [None] * 5 + list(rng.uniform(0.0, 1.0, size=100))
        counts = [O.replay_decisions(trace, 5, d) for d in (0.0, 0.1, 0.25, 0.3, 0.5, 1.0)]
        assert counts == sorted(counts, reverse=True) and counts[0] == len(trace)


@pytest.mark.parametrize("name", case_names())
def test_oracle_matches_reference_golden(name, golden_cases):
    c = golden_cases[name]
    P = c["P"]
    grads = lambda w, s, _p: O.synthetic_grad32(c["grad_seed"], w, s, P)
    init = O.init_params_linear(c["d"], c["init_seed"])
    np.testing.assert_array_equal(init, c["init"])
    res = O.simulate_selsync(
        init, c["n"], c["steps"], grads, delta=c["delta"], warmup=c["warmup"],
        smoothing=c["smoothing"], lr=c["lr"], aggregation=c["aggregation"],
        capture=lambda s: s in set(c["snap_steps"].tolist()))
    # bit-exact: same float64 operations in the same order as the reference
    np.testing.assert_array_equal(res.grad_norm_sq, c["grad_norm_sq"])
    np.testing.assert_array_equal(res.ewma, c["ewma"])
    np.testing.assert_array_equal(res.delta_g, c["delta_g"])
    assert (res.decision[:, None] == c["decision"]).all()
    np.testing.assert_array_equal(res.finals, c["finals"])
    for i, s in enumerate(c["snap_steps"]):
        np.testing.assert_array_equal(res.trajectory[int(s)], c["snaps"][i])
