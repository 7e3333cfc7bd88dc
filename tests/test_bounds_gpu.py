"""Out-of-bounds guard bands around every compute entry point.

compute-sanitizer is closed on this GPU pool, so out-of-bounds accesses are
caught the way the pool asks: every operand is a view inside a larger
allocation whose guard bands (before and after, at ragged and misaligned
offsets) hold a NaN canary. A stray WRITE changes a canary (checked
bit-for-bit); a stray READ pulls a NaN into ||g||^2 or into the update and
makes the result disagree with the float64 restatement (checked too). The
symmetric-memory step is covered through a world-1 group (its buffers are
allocated by the step; the step's own inputs -- gradient and momentum -- are
guarded).
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_07950_b200 import kernels as K  # noqa: E402

DEV = torch.device("cuda:0")
CANARY = float("nan")
GUARD = 37  # floats each side (not a multiple of 4: guards straddle 16-byte vectors)
SIZES = [1, 3, 5, 7, 1002, 4097, 65539]
OFFSETS = [0, 1, 3]


class Guarded:
    """A length-n view at `off` floats into a buffer with NaN guard bands."""

    def __init__(self, values: torch.Tensor, off: int):
        n = values.numel()
        self.buf = torch.full((GUARD + off + n + GUARD,), CANARY, device=DEV)
        self.lo, self.hi = GUARD + off, GUARD + off + n
        self.view = self.buf[self.lo:self.hi]
        self.view.copy_(values)
        self.snapshot = self.buf.clone()

    def check(self, what: str):
        torch.cuda.synchronize()
        a = self.buf.view(torch.int32)
        b = self.snapshot.view(torch.int32)
        assert torch.equal(a[: self.lo], b[: self.lo]), f"{what}: write before the view"
        assert torch.equal(a[self.hi:], b[self.hi:]), f"{what}: write after the view"


def randn(n, seed):
    return torch.randn(n, generator=torch.Generator(device=DEV).manual_seed(seed), device=DEV)


def ref_sgd(w, g, m, lr, mu, wd, nest):
    w, g = w.double(), g.double()
    d = g + wd * w
    if mu:
        m = mu * m.double() + d
        d = d + mu * m if nest else m
    return w - lr * d, m


def assert_close(got, want, what, rtol=1e-6):
    got, want = got.double(), want.double()
    assert torch.isfinite(got).all(), f"{what}: non-finite result (read a guard?)"
    tol = rtol * max(1.0, float(want.abs().max()))
    assert float((got - want).abs().max()) <= tol, what


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("off", OFFSETS)
def test_norm_and_signal_stay_in_bounds(n, off):
    g = Guarded(randn(n, n + off), off)
    ws = K.Workspace(DEV)
    sig = K.DeviceSignal(DEV, 0.5, 2, trace_capacity=8)
    want = g.view.double() @ g.view.double()
    got = K.norm_sq(g.view, ws=ws)
    assert float(got.item()) == pytest.approx(float(want), rel=1e-12)
    K.norm_signal(g.view, sig, 0.3, ws)
    assert float(sig.read_trace()["grad_norm_sq"][0]) == pytest.approx(float(want), rel=1e-12)
    g.check("K1 / K1+K2")


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("off", OFFSETS)
@pytest.mark.parametrize("mu,nest", [(0.0, False), (0.9, False), (0.9, True)])
def test_update_kernels_stay_in_bounds(n, off, mu, nest):
    w0, g0, m0 = randn(n, 1), randn(n, 2), randn(n, 3)
    want_w, _ = ref_sgd(w0, g0, m0, 0.1, mu, 1e-3, nest)
    # K3
    w, g, m = Guarded(w0, off), Guarded(g0, off), Guarded(m0, off)
    K.sgd_update_(w.view, g.view, m.view if mu else None, lr=0.1, momentum=mu, weight_decay=1e-3,
                  nesterov=nest)
    assert_close(w.view, want_w, "K3")
    for t, name in ((w, "w"), (g, "g"), (m, "m")):
        t.check(f"K3 {name}")
    # K13 (+ K2)
    w, g, m = Guarded(w0, off), Guarded(g0, off), Guarded(m0, off)
    sig = K.DeviceSignal(DEV, 0.5, 2, trace_capacity=8)
    K.update_norm_signal_(w.view, g.view, m.view if mu else None, sig, K.Workspace(DEV), lr=0.1,
                          delta=0.3, momentum=mu, weight_decay=1e-3, nesterov=nest)
    assert_close(w.view, want_w, "K13")
    assert float(sig.read_trace()["grad_norm_sq"][0]) == pytest.approx(float(g0.double() @ g0.double()),
                                                                       rel=1e-12)
    for t, name in ((w, "w"), (g, "g"), (m, "m")):
        t.check(f"K13 {name}")


def test_multi_tensor_table_stays_in_bounds():
    shapes = [1, 64, 3, 1002, 4097, 5, 65539]
    ws = [Guarded(randn(s, 10 + i), i % 4) for i, s in enumerate(shapes)]
    gs = [Guarded(randn(s, 20 + i), (i + 1) % 4) for i, s in enumerate(shapes)]
    ms = [Guarded(randn(s, 30 + i), (i + 2) % 4) for i, s in enumerate(shapes)]
    want = [ref_sgd(w.view.clone(), g.view, m.view.clone(), 0.1, 0.9, 1e-3, False)[0]
            for w, g, m in zip(ws, gs, ms)]
    flat = torch.cat([g.view for g in gs]).double()
    sig = K.DeviceSignal(DEV, 0.5, 2, trace_capacity=8)
    K.update_norm_signal_multi_([w.view for w in ws], [g.view for g in gs], [m.view for m in ms], sig,
                                K.Workspace(DEV), lr=0.1, delta=0.3, momentum=0.9, weight_decay=1e-3)
    assert float(sig.read_trace()["grad_norm_sq"][0]) == pytest.approx(float(flat @ flat), rel=1e-12)
    assert float(K.norm_sq_multi([g.view for g in gs]).item()) == pytest.approx(float(flat @ flat), rel=1e-12)
    for i, (w, g, m) in enumerate(zip(ws, gs, ms)):
        assert_close(w.view, want[i], f"K13 multi tensor {i}")
        for t, name in ((w, "w"), (g, "g"), (m, "m")):
            t.check(f"K13 multi tensor {i} {name}")


@pytest.mark.parametrize("n", [1, 5, 1002, 65539])
def test_replica_mean_stays_in_bounds(n):
    bufs = [Guarded(randn(n, 40 + r), r % 4) for r in range(3)]
    want = torch.stack([b.view.double() for b in bufs]).mean(0)
    out = Guarded(torch.zeros(n, device=DEV), 1)
    K.mean([b.view for b in bufs], out=out.view)
    assert_close(out.view, want, "mean")
    out.check("mean out")
    K.replica_average_([b.view for b in bufs])
    for r, b in enumerate(bufs):
        assert_close(b.view, want, f"replica {r}")
        b.check(f"replica {r}")


@pytest.mark.parametrize("order", ["update_first", "norm_first"])
@pytest.mark.parametrize("delta", [0.0, 1e9], ids=["sync", "local"])
def test_one_launch_step_inputs_stay_in_bounds(order, delta, tmp_path):
    import torch.distributed as dist

    from paper_2307_07950_b200 import SelSyncConfig
    from paper_2307_07950_b200.step import SelSyncStep

    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1, device_id=DEV)
    try:
        n = 66004  # norm-first needs 16-byte aligned streams (GUARD + 3 = 40 floats); ragged last tile
        w0, g0 = randn(n, 50) * 0.05, randn(n, 51)
        g, m = Guarded(g0, 3), Guarded(torch.zeros(n, device=DEV), 3)
        cfg = SelSyncConfig(delta=delta, warmup=1, momentum=0.9, weight_decay=4e-4)
        st = SelSyncStep(w0.clone(), g.view, cfg, momentum_buffer=m.view, collective="symm", order=order,
                         tile_elems=1024)
        st.step(0.01)
        st.synchronize()
        want, _ = ref_sgd(w0, g0, torch.zeros(n, device=DEV), 0.01, 0.9, 4e-4, False)  # first step: m = d
        assert_close(st.params, want, f"one-launch step {order}")
        g.check("step g")
        m.check("step m")
    finally:
        dist.destroy_process_group()
