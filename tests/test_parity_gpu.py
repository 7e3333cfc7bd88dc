"""Decision-trace / EWMA / Delta / parameter parity of the B200 SelSync step
with the CPU reference, on identical seeded fp32 gradients and parameters.

Bar (BASELINE.json north_star): identical sync/local decision trace except
steps where |Delta - delta| < 1e-6 relative; EWMA and Delta within 1e-5
relative; parameters within 1e-5 relative in fp32 after all steps. Golden
traces come from the UNMODIFIED reference (tests/golden/make_golden.py); the
momentum / weight-decay cases (not in the reference) use the oracle's
torch.optim.SGD restatement.
"""

import math

import numpy as np
import pytest
import torch

from conftest import case_names
from oracle import selsync_oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_07950_b200 import ConfigError, SelSyncConfig, SignalError  # noqa: E402
from paper_2307_07950_b200.replicas import ReplicaSelSync  # noqa: E402
from paper_2307_07950_b200.step import SelSyncStep  # noqa: E402

DEV = torch.device("cuda:0")
TIE_REL = 1e-6


def assert_trace_parity(dec_got, dec_want, deltas_want, delta, warmup):
    """Decisions identical except at ties |Delta - delta| < 1e-6 relative."""
    for s, (a, b) in enumerate(zip(dec_got, dec_want)):
        if a != b:
            row = deltas_want[s]
            tie = s >= warmup and any(
                not math.isnan(d) and abs(d - delta) <= TIE_REL * max(abs(delta), 1e-300) for d in row)
            assert tie, f"step {s}: got {'sync' if a else 'local'}, reference {'sync' if b else 'local'}"


def params_close(got, want):
    scale = np.abs(want).max()
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-5 * scale)


def run_replicas(c, fuse, cfg=None, steps=None):
    n, P, steps = c["n"], c["P"], steps or c["steps"]
    cfg = cfg or SelSyncConfig(delta=c["delta"], aggregation=c["aggregation"], warmup=c["warmup"],
                               smoothing=c["smoothing"])
    rep = ReplicaSelSync(torch.tensor(c["init"], dtype=torch.float32, device=DEV), n, cfg, fuse=fuse)
    for s in range(steps):
        rep.set_grads([torch.from_numpy(O.synthetic_grad32(c["grad_seed"], w, s, P)).to(DEV)
                       for w in range(n)])
        rep.step(c["lr"])
    torch.cuda.synchronize()
    return rep


@pytest.mark.parametrize("fuse", [True, False], ids=["fused", "prescale"])
@pytest.mark.parametrize("name", case_names())
def test_replicas_match_reference_golden(name, fuse, golden_cases):
    c = golden_cases[name]
    rep = run_replicas(c, fuse)
    steps, n = c["steps"], c["n"]
    want_dec = c["decision"][:, 0]
    assert_trace_parity(rep.decisions, want_dec, c["delta_g"], c["delta"], c["warmup"])
    for w in range(n):
        tr = rep.trace(w)[:steps]
        np.testing.assert_allclose(tr["grad_norm_sq"], c["grad_norm_sq"][:, w], rtol=1e-12)
        np.testing.assert_allclose(tr["ewma"], c["ewma"][:, w], rtol=1e-5)
        np.testing.assert_allclose(tr["delta_g"], c["delta_g"][:, w], rtol=1e-5, atol=1e-12)
        params_close(rep.params[w].double().cpu().numpy(), c["finals"][w])


@pytest.mark.parametrize("mu,wd,nest,agg", [(0.9, 4e-4, False, "params"), (0.9, 4e-4, True, "params"),
                                             (0.9, 0.0, False, "grads"), (0.0, 1e-3, False, "params")])
@pytest.mark.parametrize("fuse", [True, False], ids=["fused", "prescale"])
def test_replicas_momentum_match_oracle(mu, wd, nest, agg, fuse):
    n, d, steps, seed, delta, warmup, lam, lr = 4, 250, 40, 3, 0.02, 5, None, 0.05
    P = 2 * d + 2
    init = O.init_params_linear(d, 5).astype(np.float32).astype(np.float64)
    cfg = SelSyncConfig(delta=delta, aggregation=agg, warmup=warmup, smoothing=lam, momentum=mu,
                        weight_decay=wd, nesterov=nest)
    rep = ReplicaSelSync(torch.tensor(init, dtype=torch.float32, device=DEV), n, cfg, fuse=fuse)
    for s in range(steps):
        rep.set_grads([torch.from_numpy(O.synthetic_grad32(seed, w, s, P)).to(DEV) for w in range(n)])
        rep.step(lr)
    ref = O.simulate_selsync(init, n, steps, lambda w, s, _p: O.synthetic_grad32(seed, w, s, P),
                             delta=delta, warmup=warmup, smoothing=lam, lr=lr, aggregation=agg,
                             momentum=mu, weight_decay=wd, nesterov=nest)
    assert 0 < ref.decision.sum() < steps
    assert_trace_parity(rep.decisions, ref.decision, ref.delta_g, delta, warmup)
    for w in range(n):
        params_close(rep.params[w].double().cpu().numpy(), ref.finals[w])


@pytest.mark.parametrize("agg,fuse", [("params", True), ("params", False), ("grads", True)])
def test_single_rank_step_matches_oracle(agg, fuse):
    """SelSyncStep (the per-rank NCCL path) at world size 1."""
    d, steps, seed, delta, warmup, lr = 5000, 60, 11, 0.003, 4, 0.1
    P = 2 * d + 2
    init = O.init_params_linear(d, 2).astype(np.float32).astype(np.float64)
    w = torch.tensor(init, dtype=torch.float32, device=DEV)
    g = torch.zeros_like(w)
    step = SelSyncStep(w, g, SelSyncConfig(delta=delta, aggregation=agg, warmup=warmup,
                                           momentum=0.9, weight_decay=1e-4), fuse=fuse)
    got = []
    for s in range(steps):
        g.copy_(torch.from_numpy(O.synthetic_grad32(seed, 0, s, P)))
        got.append(step.step(lr) == "sync")
    ref = O.simulate_selsync(init, 1, steps, lambda w_, s, _p: O.synthetic_grad32(seed, 0, s, P),
                             delta=delta, warmup=warmup, lr=lr, aggregation=agg, momentum=0.9,
                             weight_decay=1e-4)
    assert 0 < ref.decision.sum() < steps
    assert_trace_parity(got, ref.decision, ref.delta_g, delta, warmup)
    recs = step.records()
    np.testing.assert_allclose([r["ewma"] for r in recs], ref.ewma[:, 0], rtol=1e-12)
    assert [r["decision"] == "sync" for r in recs] == got
    assert step.decisions() == got
    params_close(w.double().cpu().numpy(), ref.finals[0])
    st = step.signal_state()
    assert st.step_count == steps and st.ewma_current == pytest.approx(ref.states[0].ewma_current, rel=1e-12)


def test_single_rank_async_steps_match_oracle():
    """step_async: no host round-trip; decisions are read from the device ring afterwards."""
    d, steps, seed, delta, warmup, lr = 3000, 80, 13, 0.003, 4, 0.1
    P = 2 * d + 2
    init = O.init_params_linear(d, 4).astype(np.float32).astype(np.float64)
    w = torch.tensor(init, dtype=torch.float32, device=DEV)
    g = torch.zeros_like(w)
    step = SelSyncStep(w, g, SelSyncConfig(delta=delta, warmup=warmup, momentum=0.9, weight_decay=4e-4),
                       trace_capacity=64)  # ring smaller than the run: wraps
    assert step.async_capable
    host = [torch.from_numpy(O.synthetic_grad32(seed, 0, s, P)).pin_memory() for s in range(steps)]
    for s in range(steps):
        g.copy_(host[s], non_blocking=True)
        step.step_async(lr)
    step.synchronize()
    ref = O.simulate_selsync(init, 1, steps, lambda w_, s, _p: O.synthetic_grad32(seed, 0, s, P),
                             delta=delta, warmup=warmup, lr=lr, momentum=0.9, weight_decay=4e-4)
    assert 0 < ref.decision.sum() < steps
    got = step.decisions()
    assert len(got) == 64
    assert_trace_parity(got, ref.decision[-64:], ref.delta_g[-64:], delta, -1)
    params_close(w.double().cpu().numpy(), ref.finals[0])


def test_captured_steps_match_oracle():
    """SelSyncStep.capture: one CUDA graph per gradient buffer, replayed --
    the same trace and parameters as the oracle (and as eager steps)."""
    d, steps, seed, delta, warmup, lr = 3000, 40, 17, 0.003, 2, 0.1
    P = 2 * d + 2
    init = O.init_params_linear(d, 5).astype(np.float32).astype(np.float64)
    w = torch.tensor(init, dtype=torch.float32, device=DEV)
    bufs = [torch.zeros_like(w) for _ in range(steps)]
    for s in range(steps):
        bufs[s].copy_(torch.from_numpy(O.synthetic_grad32(seed, 0, s, P)))
    step = SelSyncStep(w, bufs[0], SelSyncConfig(delta=delta, warmup=warmup, momentum=0.9, weight_decay=4e-4))
    step.step_async(lr)  # the first step initialises the momentum buffer eagerly
    graphs = []
    for s in range(1, steps):
        step.grads = bufs[s]
        graphs.append(step.capture(lr))
    assert step.steps_done == 1  # capturing does not run a step
    for gr in graphs:
        gr.replay()
    step.synchronize()
    ref = O.simulate_selsync(init, 1, steps, lambda w_, s, _p: O.synthetic_grad32(seed, 0, s, P),
                             delta=delta, warmup=warmup, lr=lr, momentum=0.9, weight_decay=4e-4)
    assert 0 < ref.decision.sum() < steps
    assert_trace_parity(step.decisions(), ref.decision, ref.delta_g, delta, warmup)
    params_close(w.double().cpu().numpy(), ref.finals[0])
    with pytest.raises(ConfigError):
        SelSyncStep(w.clone(), bufs[0], SelSyncConfig(delta=delta, warmup=warmup)).capture(lr)


@pytest.mark.parametrize("per_graph", [3, 13])
def test_multi_step_graphs_match_oracle(per_graph):
    """capture(lr, grads_seq): several consecutive steps in one CUDA graph
    (programmatic dependent launch between the step kernels inside it), the
    remainder as one-step graphs -- same trace and parameters as the oracle."""
    d, steps, seed, delta, warmup, lr = 3000, 40, 17, 0.003, 2, 0.1
    P = 2 * d + 2
    init = O.init_params_linear(d, 5).astype(np.float32).astype(np.float64)
    w = torch.tensor(init, dtype=torch.float32, device=DEV)
    bufs = [torch.tensor(O.synthetic_grad32(seed, 0, s, P), dtype=torch.float32, device=DEV) for s in range(steps)]
    step = SelSyncStep(w, bufs[0], SelSyncConfig(delta=delta, warmup=warmup, momentum=0.9, weight_decay=4e-4))
    step.step_async(lr)
    graphs, s = [], 1
    while s < steps:
        k = min(per_graph, steps - s)
        graphs.append(step.capture(lr, bufs[s:s + k]))
        s += k
    assert step.steps_done == 1 and step.grads is bufs[0]
    for gr in graphs:
        gr.replay()
    step.synchronize()
    assert step.steps_done == steps
    ref = O.simulate_selsync(init, 1, steps, lambda w_, s, _p: O.synthetic_grad32(seed, 0, s, P),
                             delta=delta, warmup=warmup, lr=lr, momentum=0.9, weight_decay=4e-4)
    assert 0 < ref.decision.sum() < steps
    assert_trace_parity(step.decisions(), ref.decision, ref.delta_g, delta, warmup)
    params_close(w.double().cpu().numpy(), ref.finals[0])
    with pytest.raises(ConfigError):
        step.capture(lr, [])


@pytest.mark.parametrize("order", ["update_first", "norm_first", "adaptive"])
def test_single_rank_symmetric_step_matches_oracle(order, tmp_path):
    """The one-launch symmetric-memory step on one rank (world-1 group, the
    configuration used to profile it under ncu): same trace and parameters."""
    import torch.distributed as dist

    d, steps, seed, delta, warmup, lr = 40000, 24, 23, 0.03, 2, 0.1  # 8 local, 16 sync (4.7% from a tie)
    P = 2 * d + 2
    init = O.init_params_linear(d, 6).astype(np.float32).astype(np.float64)
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1, device_id=DEV)
    try:
        w = torch.tensor(init, dtype=torch.float32, device=DEV)
        g = torch.zeros_like(w)
        step = SelSyncStep(w, g, SelSyncConfig(delta=delta, warmup=warmup, momentum=0.9, weight_decay=4e-4),
                           collective="symm", order=order, tile_elems=4096)
        assert step.collective == "symm" and step.flag_exchange == "fused"
        for s in range(steps):
            g.copy_(torch.from_numpy(O.synthetic_grad32(seed, 0, s, P)))
            step.step_async(lr)
        step.synchronize()
        got_w = step.params.double().cpu().numpy()
        got_dec = step.decisions()
    finally:
        dist.destroy_process_group()
    ref = O.simulate_selsync(init, 1, steps, lambda w_, s, _p: O.synthetic_grad32(seed, 0, s, P),
                             delta=delta, warmup=warmup, lr=lr, momentum=0.9, weight_decay=4e-4)
    assert 0 < ref.decision.sum() < steps
    assert_trace_parity(got_dec, ref.decision, ref.delta_g, delta, warmup)
    params_close(got_w, ref.finals[0])


def test_nan_gradient_raises_signal_error():
    w = torch.zeros(1000, device=DEV)
    g = torch.ones_like(w)
    step = SelSyncStep(w, g, SelSyncConfig(delta=0.1, warmup=1), fuse=False)
    step.step(0.1)
    g[3] = float("nan")
    with pytest.raises(SignalError):
        step.step(0.1)
    assert step.signal_state().step_count == 1  # state unchanged (signal.py:67-68)


def test_device_trace_as_reference_metrics_jsonl(tmp_path, golden_cases):
    """The B200 run's trace, written in the reference's metrics.jsonl schema,
    replays to the same counterfactual sync counts as the reference's file."""
    import json
    from pathlib import Path

    from paper_2307_07950_b200 import trace as T

    c = golden_cases["n4_mixed"]
    rep = run_replicas(c, True)
    rows = T.to_metrics_rows(rep.records(), n_params=c["P"])
    out = tmp_path / "metrics.jsonl"
    T.write_metrics_jsonl(rows, out)
    mine = T.load_metrics_jsonl(out)
    gold_dir = Path(__file__).resolve().parent / "golden"
    ref = T.load_metrics_jsonl(gold_dir / "n4_mixed_metrics.jsonl")
    assert [(r["step"], r["worker_id"], r["decision"]) for r in mine] == \
           [(r["step"], r["worker_id"], r["decision"]) for r in ref]
    for a, b in zip(mine, ref):
        assert a["ewma"] == pytest.approx(b["ewma"], rel=1e-12)
        assert (a["delta_g"] is None) == (b["delta_g"] is None)
    want = json.loads((gold_dir / "n4_mixed_replay.json").read_text())
    got = T.replay_trace(mine, want["worker"], want["grid"], want["warmup"])
    assert [n for _, n in got] == want["syncs"]


def test_tensor_list_step_matches_flat_step():
    """The pointer-table K13 over separate tensors reproduces the flat path:
    same parameters (same per-element arithmetic), same norms and decisions."""
    from paper_2307_07950_b200.step import TensorListSelSyncStep

    rng = np.random.default_rng(3)
    sizes = [int(s) for s in rng.integers(1, 20000, size=150)] + [64, 3, 1 << 16]
    cfg = SelSyncConfig(delta=0.02, warmup=3, momentum=0.9, weight_decay=4e-4)
    ws = [torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(DEV) for s in sizes]
    gs = [torch.zeros_like(w) for w in ws]
    flat_w = torch.cat([w.clone() for w in ws])
    flat_g = torch.zeros_like(flat_w)
    a = TensorListSelSyncStep(ws, gs, cfg)
    b = SelSyncStep(flat_w, flat_g, cfg)
    for s in range(16):
        g_all = torch.from_numpy(O.synthetic_grad32(5, 0, s, flat_w.numel())).to(DEV)
        flat_g.copy_(g_all)
        for g, part in zip(gs, torch.split(g_all, sizes)):
            g.copy_(part)
        assert a.step(0.05) == b.step(0.05)
    torch.testing.assert_close(torch.cat(ws), flat_w, rtol=0, atol=0)
    ra, rb = a.signal.read_trace()[:16], b.signal.read_trace()[:16]
    np.testing.assert_allclose(ra["grad_norm_sq"], rb["grad_norm_sq"], rtol=1e-12)
    assert 0 < sum(a.decision_log) < 16


_PDL_SCRIPT = r"""
import hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2307_07950_b200 import SelSyncConfig
from paper_2307_07950_b200.step import SelSyncStep
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev).manual_seed(5)
h = hashlib.sha256()
for P in (1_002, 1_000_003):
    w = (torch.rand(P, generator=gen, device=dev) - 0.5) * 0.1
    grads = [torch.randn(P, generator=gen, device=dev) * s for s in (1.0, 1.0, 1.5, 1.5, 0.7)]
    st = SelSyncStep(w, grads[0], SelSyncConfig(delta=0.2, warmup=2, smoothing=0.5, momentum=0.9,
                                                weight_decay=4e-4))
    for k in range(40):  # back to back: consecutive launches overlap under PDL
        st.grads = grads[k % 5]
        st.step_async(0.05)
    st.synchronize()
    for t in (st.params, st.momentum, st.signal.trace[: 32 * 40]):
        h.update(t.cpu().numpy().tobytes())
    h.update(bytes(st.decisions()))
print(h.hexdigest())
"""


def test_programmatic_dependent_launch_changes_no_bit():
    """Back-to-back steps launched with programmatic stream serialization
    (the default) and without it (SS_PDL=0) give bit-identical parameters,
    momentum, trace rows and decisions: no kernel touches memory before
    griddepcontrol.wait returns."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    out = {}
    for pdl in ("1", "0"):
        p = subprocess.run([sys.executable, "-c", _PDL_SCRIPT, root], capture_output=True, text=True, timeout=300,
                           env={**os.environ, "SS_PDL": pdl})
        assert p.returncode == 0, p.stderr[-2000:]
        out[pdl] = p.stdout.strip().splitlines()[-1]
    assert out["1"] == out["0"]
