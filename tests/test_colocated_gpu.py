"""The multi-rank step kernels on ONE GPU: N colocated ranks (same-device
peer buffers, the N grids as slices of one cooperative launch)
against the reference's golden N-worker traces and the float64 oracle.

These run the W = 2 / 4 / 8 instantiations of ``step_kernel`` /
``step_ga_kernel`` -- the seq-tagged vote exchange (runtime.py:319-333), the
conditional mean with 1/N in the epilogue (runtime.py:275-294 ->
strategies.py:159-168), the norm-first tile tickets, the known-sync pass, the
NaN paths and the bootstrap broadcast (runtime.py:178-191) -- on a
single-GPU box. Bar (BASELINE.json north_star): decisions identical except at
|Delta - delta| < 1e-6 relative ties, EWMA / Delta within 1e-5 relative,
parameters within 1e-5 relative after all steps.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import case_names
from oracle import selsync_oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_07950_b200 import ConfigError, SelSyncConfig, SignalError  # noqa: E402
from paper_2307_07950_b200.colocated import ColocatedSelSync  # noqa: E402
from test_parity_gpu import assert_trace_parity, params_close  # noqa: E402

DEV = torch.device("cuda:0")
ORDERS = ["update_first", "norm_first", "adaptive", "nan_safe"]
MULTI = [n for n in case_names() if not n.startswith("n1_")]

sys.path.insert(0, str(Path(__file__).resolve().parent))
import mp_selsync_worker as MW  # noqa: E402


def run_case(c, order, tile_elems=None, async_every=1):
    n, P = c["n"], c["P"]
    cfg = SelSyncConfig(delta=c["delta"], aggregation=c["aggregation"], warmup=c["warmup"],
                        smoothing=c["smoothing"])
    col = ColocatedSelSync(torch.tensor(c["init"], dtype=torch.float32, device=DEV), n, cfg, order=order,
                           tile_elems=tile_elems, timeout_s=5.0)
    host = [[torch.from_numpy(O.synthetic_grad32(c["grad_seed"], r, s, P)).pin_memory() for r in range(n)]
            for s in range(c["steps"])]
    for s in range(c["steps"]):
        col.set_grads([h.to(DEV, non_blocking=True) for h in host[s]])
        col.step(c["lr"])
        if async_every and s % async_every == 0:
            col.synchronize()
    col.synchronize()
    return col


def check_golden(col, c):
    n, steps = c["n"], c["steps"]
    for r in range(n):
        assert_trace_parity(col.decisions(r), c["decision"][:, 0], c["delta_g"], c["delta"], c["warmup"])
        tr = col.trace(r)[:steps]
        np.testing.assert_allclose(tr["grad_norm_sq"], c["grad_norm_sq"][:, r], rtol=1e-12)
        np.testing.assert_allclose(tr["ewma"], c["ewma"][:, r], rtol=1e-5)
        np.testing.assert_allclose(tr["delta_g"], c["delta_g"][:, r], rtol=1e-5, atol=1e-12)
        params_close(col.params[r].double().cpu().numpy(), c["finals"][r])


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("name", MULTI)
def test_colocated_ranks_match_reference_golden(name, order, golden_cases):
    """Every multi-worker golden trace of the unmodified reference (N = 2, 4,
    8; parameter and gradient aggregation; delta = 0, 1e9, mixed) through the
    one-launch step kernel of each rank, one tile per buffer."""
    c = golden_cases[name]
    if c["aggregation"] == "grads" and order != "adaptive":
        pytest.skip("gradient aggregation has one order (step_ga_kernel)")
    col = run_case(c, order, async_every=0)
    check_golden(col, c)


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("name", ["cfg0_n2_d0.3", "n4_mixed", "n8_mixed", "n4_delta0", "n4_grads"])
def test_colocated_many_small_tiles(name, order, golden_cases):
    """Same traces with 64-element tiles: several tiles per rank, lag groups,
    owners t mod N, a ragged last tile and a scalar tail (P = 1002 / 402 /
    202 / 602), and a host sync every 7 steps (ranks restart together)."""
    c = golden_cases[name]
    if c["aggregation"] == "grads" and order != "adaptive":
        pytest.skip("gradient aggregation has one order (step_ga_kernel)")
    col = run_case(c, order, tile_elems=64, async_every=7)
    check_golden(col, c)


@pytest.fixture(scope="module")
def large_oracle():
    """Oracle run of mp_selsync_worker.LARGE per world size (float64 numpy)."""
    cache = {}

    def get(n, aggregation, delta):
        key = (n, aggregation, delta)
        if key not in cache:
            c = MW.LARGE
            init = MW.large_init(c["seed"], c["P"]).astype(np.float64)
            cache[key] = O.simulate_selsync(
                init, n, c["steps"],
                lambda w, s, _p: O.synthetic_grad32(c["seed"], w, s, c["P"]).astype(np.float64),
                delta=delta, warmup=c["warmup"], smoothing=c["smoothing"], lr=c["lr"], momentum=c["momentum"],
                weight_decay=c["weight_decay"], aggregation=aggregation)
        return cache[key]
    return get


LARGE_VARIANTS = ["update_first", "norm_first", "adaptive", "nan_safe", "bsp", "ga"]


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("variant", LARGE_VARIANTS)
def test_colocated_large_ragged_matches_oracle(n, variant, large_oracle):
    """P = 1,000,003 in 4096-element tiles (245 tiles, a 3-element scalar
    tail), momentum + weight decay, mixed decisions (bsp: delta = 0, every
    step the known-sync pass; ga: gradient aggregation) at W = 2, 4, 8."""
    c = MW.LARGE
    P = c["P"]
    agg = "grads" if variant == "ga" else "params"
    delta = 0.0 if variant == "bsp" else c["delta"]
    order = "adaptive" if variant in ("bsp", "ga") else variant
    cfg = SelSyncConfig(delta=delta, warmup=c["warmup"], smoothing=c["smoothing"], momentum=c["momentum"],
                        weight_decay=c["weight_decay"], aggregation=agg)
    col = ColocatedSelSync(torch.from_numpy(MW.large_init(c["seed"], P)).to(DEV), n, cfg, order=order,
                           tile_elems=c["tile"], timeout_s=10.0)
    for s in range(c["steps"]):
        col.set_grads([torch.from_numpy(O.synthetic_grad32(c["seed"], r, s, P)).to(DEV) for r in range(n)])
        col.step(c["lr"])
    col.synchronize()
    ref = large_oracle(n, agg, delta)
    for r in range(n):
        dec = col.decisions(r)
        assert_trace_parity(dec, ref.decision, ref.delta_g, delta, c["warmup"])
        recs = col.ranks[r].records()
        np.testing.assert_allclose([x["ewma"] for x in recs], ref.ewma[:, r], rtol=1e-5)
        params_close(col.params[r].double().cpu().numpy(), ref.finals[r])
    if variant == "bsp":
        assert all(dec), "delta = 0 must sync every step"
    else:
        assert 0 < sum(dec[c["warmup"]:]) < c["steps"] - c["warmup"], "case must mix sync and local steps"


@pytest.mark.parametrize("n", [1, 2, 8])
def test_known_pass_one_tile_many_blocks(n):
    """The known-sync pass with ONE tile and a wide grid: the tile (and K2,
    which advances step_count) can finish before late blocks of the same
    launch have read step_count to pick the order. Every block must take the
    same snapshot (K2 waits for all of them), else a late block runs the
    norm sweep of a step the others skipped and every later ||g||^2 is wrong.
    Warmup 6 (known), then mixed steps: trace and parameters vs the oracle."""
    P, steps, seed, warmup, delta, lr = 1 << 18, 14, 31, 6, 0.02, 0.05
    init = O.init_params_linear((P - 2) // 2, 9).astype(np.float32).astype(np.float64)
    cfg = SelSyncConfig(delta=delta, warmup=warmup, smoothing=0.5, momentum=0.9, weight_decay=4e-4)
    col = ColocatedSelSync(torch.tensor(init, dtype=torch.float32, device=DEV), n, cfg, order="adaptive",
                           tile_elems=P, timeout_s=5.0)
    assert col.blocks_per_rank >= 64
    for s in range(steps):
        col.set_grads([torch.from_numpy(O.synthetic_grad32(seed, r, s, P)).to(DEV) for r in range(n)])
        col.step(lr)
    col.synchronize()
    ref = O.simulate_selsync(init, n, steps, lambda w, s, _p: O.synthetic_grad32(seed, w, s, P), delta=delta,
                             warmup=warmup, smoothing=0.5, lr=lr, momentum=0.9, weight_decay=4e-4)
    for r in range(n):
        tr = col.trace(r)[:steps]
        np.testing.assert_allclose(tr["grad_norm_sq"], ref.grad_norm_sq[:, r], rtol=1e-12)
        assert_trace_parity(col.decisions(r), ref.decision, ref.delta_g, delta, warmup)
        params_close(col.params[r].double().cpu().numpy(), ref.finals[r])


def _nan_run(n, order, agg, warmup, nan_rank=1, P=40_000, tile=4096):
    cfg = SelSyncConfig(delta=0.05, warmup=warmup, smoothing=0.5, momentum=0.9, weight_decay=4e-4,
                        aggregation=agg)
    init = torch.from_numpy(np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)).to(DEV)
    col = ColocatedSelSync(init, n, cfg, order=order, tile_elems=tile, timeout_s=5.0)
    for s in range(3):
        col.set_grads([torch.from_numpy(O.synthetic_grad32(5, r, s, P)).to(DEV) for r in range(n)])
        col.step(0.05)
    col.synchronize()
    before = [p.clone() for p in col.params]
    moms = [st.momentum.clone() for st in col.ranks]
    grads = [torch.from_numpy(O.synthetic_grad32(5, r, 3, P)).to(DEV) for r in range(n)]
    grads[nan_rank][P // 2 + 11] = float("nan")  # a tile in the middle
    col.set_grads(grads)
    col.step(0.05)
    with pytest.raises(SignalError):
        col.synchronize()
    return col, before, moms


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("agg,order", [("params", "nan_safe"), ("grads", "adaptive")])
def test_nan_step_changes_nothing_anywhere(n, agg, order):
    """NaN-safe orders (the reference raises in observe before sgd_step,
    signal.py:67-68 / strategies.py:286 vs :383; GA defers the update after
    the exchange, :395-399): a NaN norm on one rank raises SignalError on
    every rank and leaves every rank's parameters and momentum bit-identical."""
    col, before, moms = _nan_run(n, order, agg, warmup=2)
    for r in range(n):
        assert torch.equal(col.params[r], before[r]), f"rank {r} parameters changed"
        assert torch.equal(col.ranks[r].momentum, moms[r]), f"rank {r} momentum changed"


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("order,warmup", [("update_first", 2), ("norm_first", 2), ("adaptive", 2),
                                          ("adaptive", 10)])
def test_nan_never_reaches_healthy_ranks(n, order, warmup):
    """Fused orders update before the norm is known, so the rank that met the
    NaN keeps NaN elements; no other rank may: the vote stops the mean, and in
    the known-sync pass (warmup 10: the mean runs before the vote) the poison
    tag of the NaN tile stops every later mean ticket."""
    col, before, _ = _nan_run(n, order, "params", warmup=warmup)
    for r in range(n):
        if r != 1:
            assert bool(torch.isfinite(col.params[r]).all()), f"NaN reached rank {r} ({order})"


def test_nan_safe_step_then_training_continues_after_error():
    """After SignalError the device state of every rank is still consistent:
    the NaN rank's signal state is unchanged (test_signal.py:72-76)."""
    col, _, _ = _nan_run(2, "nan_safe", "params", warmup=2)
    assert col.ranks[1].signal_state().step_count == 3
    assert col.ranks[0].signal_state().step_count == 4


def test_steps_with_a_busy_device_stay_correct():
    """Cooperative launch: while a long GEMM stream occupies SMs, each rank's
    step grid is placed whole (or waits), never partly -- the spinning blocks
    never starve the rest of their grid. Parity must hold and no timeout."""
    c = MW.LARGE
    n, P = 2, c["P"]
    cfg = SelSyncConfig(delta=c["delta"], warmup=c["warmup"], smoothing=c["smoothing"], momentum=c["momentum"],
                        weight_decay=c["weight_decay"])
    col = ColocatedSelSync(torch.from_numpy(MW.large_init(c["seed"], P)).to(DEV), n, cfg, order="adaptive",
                           tile_elems=c["tile"], timeout_s=10.0)
    side = torch.cuda.Stream(DEV)
    a = torch.randn(4096, 4096, device=DEV)
    for s in range(c["steps"]):
        with torch.cuda.stream(side):
            for _ in range(4):
                a = torch.tanh(a @ a * 1e-3)
        col.set_grads([torch.from_numpy(O.synthetic_grad32(c["seed"], r, s, P)).to(DEV) for r in range(n)])
        col.step(c["lr"])
    col.synchronize()
    side.synchronize()
    init = MW.large_init(c["seed"], P).astype(np.float64)
    ref = O.simulate_selsync(init, n, c["steps"], lambda w, s, _p: O.synthetic_grad32(c["seed"], w, s, P),
                             delta=c["delta"], warmup=c["warmup"], smoothing=c["smoothing"], lr=c["lr"],
                             momentum=c["momentum"], weight_decay=c["weight_decay"])
    for r in range(n):
        assert_trace_parity(col.decisions(r), ref.decision, ref.delta_g, c["delta"], c["warmup"])
        params_close(col.params[r].double().cpu().numpy(), ref.finals[r])


def test_plan_splits_the_device_and_ranks_cannot_launch_alone():
    """The N grids are one cooperative launch of N x G blocks (G capped so
    all fit at once); a colocated rank never launches by itself (its kernel
    would wait for peers that nothing guarantees to be running)."""
    cfg = SelSyncConfig(delta=0.05, warmup=2)
    col = ColocatedSelSync(torch.zeros(1 << 22, device=DEV), 4, cfg, order="update_first", timeout_s=2.0)
    sms = torch.cuda.get_device_properties(DEV).multi_processor_count
    assert 1 <= col.blocks_per_rank and 4 * col.blocks_per_rank <= 8 * sms
    col.step(0.1)
    col.synchronize()
    with pytest.raises(ConfigError):
        col.ranks[1].step_async(0.1)
    with pytest.raises(ConfigError):
        ColocatedSelSync(torch.zeros(8, device=DEV), 3, cfg)
    small = ColocatedSelSync(torch.zeros(1 << 22, device=DEV), 2, cfg, max_blocks=7)
    assert small.blocks_per_rank == 7
    small.step(0.1)
    small.synchronize()


def test_colocated_captured_steps_match_eager():
    """The colocated launch captured as a CUDA graph (a cooperative kernel
    node) and replayed: same decisions and parameters as eager steps."""
    n, P, steps = 2, 262_144, 10
    cfg = SelSyncConfig(delta=0.05, warmup=2, smoothing=0.5, momentum=0.9, weight_decay=4e-4)
    init = torch.from_numpy(MW.large_init(3, P)).to(DEV)
    grads = [[torch.from_numpy(O.synthetic_grad32(3, r, s, P)).to(DEV) for r in range(n)] for s in range(steps)]

    def run(capture):
        col = ColocatedSelSync(init, n, cfg, order="adaptive", tile_elems=4096, timeout_s=5.0)
        col.set_grads(grads[0])
        col.step(0.05)
        graph = col.capture(0.05) if capture else None
        for s in range(1, steps):
            col.set_grads(grads[s])
            if capture:
                graph.replay()
            else:
                col.step(0.05)
        col.synchronize()
        return col

    a, b = run(False), run(True)
    for r in range(n):
        assert a.decisions(r) == b.decisions(r)
        torch.testing.assert_close(a.params[r], b.params[r], rtol=0, atol=0)
    assert 0 < sum(a.decisions(0)[2:]) < steps - 2


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("order,agg", [("norm_first", "params"), ("adaptive", "params")])
def test_early_vote_fires_on_upward_jumps_and_changes_nothing(n, order, agg):
    """Exact early vote (norm-first orders): a block whose running lower bound
    of ||g||^2 proves the vote sync posts an early tag and the mean tickets
    start before the sweep ends. Gradients scaled [1, 1, 1.5, 1.5] cycled
    (smoothing 1, delta 0.3: local / up / local / down): the tag must appear on
    upward sync steps only, never on local steps, and the run must be
    bit-identical to the same run with the early vote off (and match the
    float64 oracle)."""
    P, steps, seed, lr = 1 << 20, 16, 41, 0.05
    scales = [1.0, 1.0, 1.5, 1.5]
    cfg = SelSyncConfig(delta=0.3, warmup=1, smoothing=1.0, momentum=0.9, weight_decay=4e-4, aggregation=agg)
    init = torch.from_numpy(MW.large_init(seed, P)).to(DEV)
    base = [torch.from_numpy(O.synthetic_grad32(seed, r, 0, P)).to(DEV) for r in range(n)]

    def run(early):
        col = ColocatedSelSync(init, n, cfg, order=order, tile_elems=16384, timeout_s=10.0, early_vote=early)
        fired = []
        for s in range(steps):
            col.set_grads([b * scales[s % 4] for b in base])
            col.step(lr)
            col.synchronize()
            tags = col.world.pads[:, 4 * n:5 * n].cpu()
            fired.append(bool((tags == s + 1).any()))
        return col, fired

    on, fired = run(True)
    off, fired_off = run(False)
    dec = on.decisions(0)
    assert not any(fired_off)
    assert any(fired), "no early vote on an upward jump"
    for s in range(steps):
        if fired[s]:
            assert dec[s] == 1 and scales[s % 4] > scales[(s - 1) % 4], (s, dec)
    for r in range(n):
        assert on.decisions(r) == off.decisions(r)
        torch.testing.assert_close(on.params[r], off.params[r], rtol=0, atol=0)
        torch.testing.assert_close(on.ranks[r].momentum, off.ranks[r].momentum, rtol=0, atol=0)
    ref = O.simulate_selsync(init.double().cpu().numpy(), n, steps,
                             lambda w, s, _p: (base[w].cpu().numpy() * np.float32(scales[s % 4])).astype(np.float64),
                             delta=0.3, warmup=1, smoothing=1.0, lr=lr, momentum=0.9, weight_decay=4e-4,
                             aggregation=agg)
    assert_trace_parity(dec, ref.decision, ref.delta_g, 0.3, 1)
    params_close(on.params[0].double().cpu().numpy(), ref.finals[0])
