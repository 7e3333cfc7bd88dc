"""Real multi-GPU SelSync over NCCL (one process per GPU, torchrun) vs the
reference's golden traces. Needs >= 2 GPUs on one box (gpurun --gpus 2/4);
skipped otherwise -- the single-GPU suite covers N workers with ReplicaSelSync."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from test_parity_gpu import assert_trace_parity, params_close  # noqa: F401

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = Path(__file__).resolve().parents[1]
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def run_torchrun(n, name, mode, out):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29533",
           str(ROOT / "tests" / "mp_selsync_worker.py"), name, mode, str(out)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                          env={**os.environ, "NCCL_DEBUG": "WARN"})
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("name,n", [("n2_lam0.5", 2), ("cfg0_n2_d0.3", 2), ("n2_grads", 2), ("n4_mixed", 4),
                                    ("n4_grads", 4), ("n8_mixed", 8)])
@pytest.mark.parametrize("mode", ["fused", "prescale", "symm-nccl", "symm-p2p", "symm-fused",
                                  "symm-normfirst", "symm-adaptive", "symm-nansafe"])
def test_nccl_ranks_match_reference(name, n, mode, tmp_path, golden_cases):
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs")
    run_torchrun(n, name, mode, tmp_path)
    c = golden_cases[name]
    for rank in range(n):
        z = np.load(tmp_path / f"{name}_{mode}_rank{rank}.npz")
        assert_trace_parity(z["decisions"], c["decision"][:, 0], c["delta_g"], c["delta"], c["warmup"])
        np.testing.assert_allclose(z["ewma"], c["ewma"][:, rank], rtol=1e-5)
        np.testing.assert_allclose(z["delta_g"], c["delta_g"][:, rank], rtol=1e-5, atol=1e-12)
        params_close(z["params"], c["finals"][rank])


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode", ["symm-adaptive", "symm-known", "symm-update-first", "symm-nansafe", "nccl",
                                  "nccl-nansafe"])
def test_nan_on_one_rank_raises_everywhere(mode, tmp_path):
    """SignalError on every rank; the NaN never reaches a healthy rank; in the
    NaN-safe orders no rank's parameters or momentum change."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29534",
           str(ROOT / "tests" / "mp_selsync_worker.py"), "nan", mode, str(tmp_path)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    for r in range(2):
        z = np.load(tmp_path / f"nan_{mode}_rank{r}.npz")
        assert bool(z["raised"])
        if r != 1:
            assert bool(z["finite"]), f"the NaN reached rank {r}"
        if mode.endswith("nansafe"):
            assert bool(z["unchanged"]), f"rank {r} changed on a NaN step"


@pytest.fixture(scope="module")
def large_oracle():
    """Oracle run of mp_selsync_worker.LARGE per world size (float64 numpy)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import mp_selsync_worker as MW
    from oracle import selsync_oracle as O

    c = MW.LARGE
    cache = {}

    def get(n, aggregation, delta):
        if (n, aggregation, delta) not in cache:
            init = MW.large_init(c["seed"], c["P"]).astype(np.float64)
            cache[n, aggregation, delta] = O.simulate_selsync(
                init, n, c["steps"], lambda w, s, _p: O.synthetic_grad32(c["seed"], w, s, c["P"]).astype(np.float64),
                delta=delta, warmup=c["warmup"], smoothing=c["smoothing"], lr=c["lr"], momentum=c["momentum"],
                weight_decay=c["weight_decay"], aggregation=aggregation)
        return cache[n, aggregation, delta]
    return get


@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("variant", ["nccl", "update_first", "norm_first", "adaptive", "p2p-mean", "nvls-mean",
                                     "two-launch", "ga", "ga-nccl", "bsp", "nan_safe", "nccl-nansafe"])
def test_large_ragged_many_tiles_match_oracle(n, variant, tmp_path, large_oracle):
    """P = 1,000,003 in 4096-element tiles, momentum + weight decay, mixed
    decisions: the tile tickets, lag groups, scalar tail and every back end
    against the float64 oracle (decisions exact but for ties, params 1e-5)."""
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29535",
           str(ROOT / "tests" / "mp_selsync_worker.py"), "large", variant, str(tmp_path)]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
    import mp_selsync_worker as MW

    delta = MW.large_delta(variant)
    ref = large_oracle(n, MW.large_aggregation(variant), delta)
    for rank in range(n):
        z = np.load(tmp_path / f"large_{variant}_rank{rank}.npz")
        assert_trace_parity(z["decisions"], ref.decision, ref.delta_g, delta, MW.LARGE["warmup"])
        np.testing.assert_allclose(z["ewma"], ref.ewma[:, rank], rtol=1e-5)
        params_close(z["params"], ref.finals[rank])
    if variant == "bsp":  # every step takes the known-sync pass (no norm sweep, no vote wait)
        assert bool(np.all(z["decisions"])), "delta = 0 must sync every step"
    else:
        assert 0 < int(np.sum(z["decisions"][MW.LARGE["warmup"]:])) < MW.LARGE["steps"] - MW.LARGE["warmup"], \
            "case must mix sync and local steps"
