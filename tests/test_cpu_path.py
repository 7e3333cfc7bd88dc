"""The CPU baseline (oracle/cpu_path.py, timed by bench.py) computes exactly
the reference step it claims to time: same decisions and parameters as the
oracle's N-worker restatement, whatever the thread slicing."""

import numpy as np
import pytest

from oracle import selsync_oracle as O
from oracle.cpu_path import CpuSelSync


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_cpu_path_matches_oracle(threads):
    n, P, steps = 3, 1001, 9
    cpu = CpuSelSync(n, P, delta=0.3, warmup=1, smoothing=1.0, momentum=0.9, weight_decay=4e-4,
                     sync_pattern=[1.0, 1.0, 1.5, 1.5], grad_ring=4, threads=threads)
    init = cpu.params[0].copy()
    ring = [[g.copy() for g in cpu.ring[w]] for w in range(n)]
    dec = [cpu.step(0.1) for _ in range(steps)]
    cpu.close()
    ref = O.simulate_selsync(init, n, steps, lambda w, s, _p: ring[w][s % 4], delta=0.3, warmup=1,
                             smoothing=1.0, lr=0.1, momentum=0.9, weight_decay=4e-4)
    assert dec == list(ref.decision)
    assert 0 < sum(dec) < steps
    for w in range(n):
        np.testing.assert_allclose(cpu.params[w], ref.finals[w], rtol=1e-12, atol=1e-15)
