"""Model-config callers (BASELINE configs 1-3): gradients of stock PyTorch
backward land in the flat buffer, the hot path sees exactly that buffer, and
the device decision trace replays bit-for-bit through the CPU oracle's
signal rules on the recorded ||g||^2 series."""

import math

import numpy as np
import pytest
import torch

from oracle import selsync_oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_07950_b200 import workloads as W  # noqa: E402
from paper_2307_07950_b200.train import SelSyncTrainer  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.mark.parametrize("name,P", [("resnet101", 42_520_650), ("vgg11", 129_176_036),
                                    ("transformer", 107_845_735)])
def test_workload_trace_replays_through_oracle(name, P):
    wl = W.build(name, DEV)
    assert W.parameter_count(wl.model) == P
    tr = SelSyncTrainer(wl, delta=0.05, warmup=3, smoothing=0.5)
    assert tr.flat.n_real == P
    norms = []
    for it in range(8):
        loss = tr.forward_backward()
        assert torch.isfinite(loss)
        # the flat buffer IS the model's gradient storage
        p0 = tr.flat.parameters[0]
        assert p0.grad.data_ptr() == tr.flat.grads.data_ptr()
        norms.append(float(torch.dot(tr.flat.grads.double(), tr.flat.grads.double())))
        tr.step.step(wl.lr(it))
        tr.iteration += 1
    recs = tr.step.records()
    got = np.array([r["grad_norm_sq"] for r in recs])
    np.testing.assert_allclose(got, norms, rtol=1e-11)
    # replay the device's own norms through the oracle's signal rules: EWMA, Delta
    # and votes must match bit-for-bit (same IEEE operations)
    st = O.SignalState(smoothing=0.5, warmup=3)
    for r in recs:
        st = O.observe(st, r["grad_norm_sq"])
        assert r["ewma"] == st.ewma_current
        if st.step_count >= 2:
            assert r["delta_g"] == O.relative_change(st)
        assert r["vote"] == (O.decide(st, 0.05) == "sync")
        assert r["decision"] == ("sync" if r["vote"] else "local")  # one rank: agreed == own


def test_channels_last_views_and_update():
    wl = W.build("resnet101", DEV)
    tr = SelSyncTrainer(wl, delta=1e9, warmup=1)
    conv = wl.model.conv1.weight
    assert conv.is_contiguous(memory_format=torch.channels_last)
    assert conv.grad.is_contiguous(memory_format=torch.channels_last)
    before = tr.flat.params.clone()
    tr.train_step(wait=True)
    g = tr.flat.grads
    # plain check of the fused update on the first step (momentum buffer seeded with d)
    d = g + wl.weight_decay * before
    want = before - wl.lr(0) * d
    torch.testing.assert_close(tr.flat.params, want, rtol=1e-5, atol=1e-6)
    assert math.isfinite(float(tr.flat.params.abs().max()))


def test_graph_replay_matches_eager():
    """fwd + bwd + SelSync step captured in one CUDA graph == the eager loop."""
    import copy

    wl = W.build("resnet101", DEV, seed=3)
    wl2 = W.build("resnet101", DEV, seed=3)
    wl2.model.load_state_dict(copy.deepcopy(wl.model.state_dict()))
    x, y = wl.make_batch(0)
    eager = SelSyncTrainer(wl, delta=0.05, warmup=2, smoothing=0.5)
    graphed = SelSyncTrainer(wl2, delta=0.05, warmup=2, smoothing=0.5)
    torch.backends.cudnn.deterministic = True
    try:
        for _ in range(3):
            eager.train_step((x, y))
        graphed.capture((x.clone(), y.clone()), warmup_iters=3)
        for _ in range(4):
            eager.train_step((x, y))
            graphed.replay_step()
        torch.cuda.synchronize()
        ra, rb = eager.step.records(), graphed.step.records()
        assert [r["decision"] for r in ra] == [r["decision"] for r in rb]
        np.testing.assert_allclose([r["grad_norm_sq"] for r in ra], [r["grad_norm_sq"] for r in rb], rtol=1e-4)
        torch.testing.assert_close(eager.flat.params, graphed.flat.params, rtol=1e-4, atol=1e-5)
    finally:
        torch.backends.cudnn.deterministic = False


def test_trainer_metrics_rows_fill_loss_and_duration(tmp_path):
    """SelSyncTrainer's metrics rows carry the loss and the step's device
    time like the reference's MetricsRecord (strategies.py:326-339,
    metrics.py:23-48), eager and graph-replayed iterations alike."""
    from paper_2307_07950_b200 import trace as T

    wl = W.build("resnet101", DEV, seed=5)
    tr = SelSyncTrainer(wl, delta=0.05, warmup=2, smoothing=0.5)
    x, y = wl.make_batch(0)
    losses = [float(tr.train_step((x, y), wait=True)[0]) for _ in range(3)]
    tr.capture((x.clone(), y.clone()), warmup_iters=2)
    losses += [float("nan")] * 2  # the capture warm-up iterations ran on a side stream
    for _ in range(3):
        losses.append(float(tr.replay_step()))
    rows = tr.metrics_rows()
    assert [r["step"] for r in rows] == list(range(8))
    for i, r in enumerate(rows):
        assert set(r) == set(T.FIELDS)
        assert r["step_duration"] > 0.0
        assert r["lr"] == pytest.approx(wl.lr(i))
        if not math.isnan(losses[i]):
            assert r["loss"] == pytest.approx(losses[i], rel=1e-6)
        assert math.isfinite(r["loss"])
    out = tmp_path / "metrics.jsonl"
    T.write_metrics_jsonl(rows, out)
    back = T.load_metrics_jsonl(out)
    assert [b["loss"] for b in back] == pytest.approx([r["loss"] for r in rows])
