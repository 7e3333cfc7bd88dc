"""sm_100a kernels vs the float64 CPU oracle, called through the C-ABI.

Tolerances: ||g||^2 is accumulated in fp64 from exact fp32 squares, so it
differs from numpy's float64 dot only by summation order (rel 1e-12). The
signal step K2 rounds exactly like Python floats (bit-exact on the same
input). Parameter updates run in fp32: rel 1e-6 per step vs the float64
oracle (atol scaled to the vector's magnitude for entries that cancel).
"""

import math

import numpy as np
import pytest
import torch

from oracle import selsync_oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_07950_b200 import kernels as K  # noqa: E402
from paper_2307_07950_b200 import _native as N  # noqa: E402
from paper_2307_07950_b200.errors import ConfigError  # noqa: E402

DEV = torch.device("cuda:0")


def rand32(n, seed, scale=1.0):
    return (np.random.default_rng(seed).standard_normal(n, dtype=np.float32) * np.float32(scale))


def dev_view(host32, offset):
    """Device copy of host32 starting `offset` floats into a larger buffer
    (to exercise misaligned heads/tails)."""
    buf = torch.zeros(host32.size + offset + 8, dtype=torch.float32, device=DEV)
    v = buf[offset: offset + host32.size]
    v.copy_(torch.from_numpy(host32))
    return v


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 7, 1002, 4097, 1 << 20, 10_000_019])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_norm_sq_matches_oracle(n, offset):
    g = rand32(n, n + offset)
    out = K.norm_sq(dev_view(g, offset))
    want = O.norm_sq(g.astype(np.float64))
    got = float(out.item())
    assert got == pytest.approx(want, rel=1e-12, abs=0.0)


def test_norm_sq_deterministic_and_scale_exact():
    g = torch.from_numpy(rand32(3_000_001, 5)).to(DEV)
    a = K.norm_sq(g).item()
    b = K.norm_sq(g).item()
    assert a == b  # fixed-order two-pass finish: bitwise reproducible
    assert K.norm_sq(g * 2).item() == 4 * a  # power-of-two scaling is exact


def test_norm_sq_multi_tensor_table():
    rng = np.random.default_rng(0)
    sizes = [int(s) for s in rng.integers(1, 5000, size=300)] + [64, 1 << 18, 3]  # > 256 tensors
    hosts = [rand32(s, i) for i, s in enumerate(sizes)]
    tensors = [dev_view(h, i % 4) for i, h in enumerate(hosts)]
    got = K.norm_sq_multi(tensors).item()
    want = O.norm_sq(np.concatenate(hosts).astype(np.float64))
    assert got == pytest.approx(want, rel=1e-12)


def test_signal_kernel_bit_exact_vs_oracle():
    rng = np.random.default_rng(4)
    xs = rng.uniform(0.5, 3.0, size=120) * np.exp(rng.normal(0, 1, size=120))
    xs[[10, 11]] = 0.0  # 0/0 -> 0 then x/0 -> inf handled below
    lam, warmup, delta = 0.08, 5, 0.02
    sig = K.DeviceSignal(DEV, lam, warmup, trace_capacity=256)
    x_dev = torch.empty(1, dtype=torch.float64, device=DEV)
    st = O.SignalState(smoothing=lam, warmup=warmup)
    for i, x in enumerate(xs):
        x_dev.fill_(float(x))
        K.signal_step(sig, x_dev, delta)
        st = O.observe(st, x)
        assert int(sig.word.item()) == (1 if O.decide(st, delta) == "sync" else 0)
    tr = sig.read_trace()[: xs.size]
    s = sig.read_state()
    assert s["ewma_current"] == st.ewma_current and s["ewma_previous"] == st.ewma_previous
    assert s["max_delta_seen"] == st.max_delta_seen and s["step_count"] == st.step_count
    np.testing.assert_array_equal(tr["grad_norm_sq"], xs)
    np.testing.assert_array_equal(tr["step"], np.arange(xs.size))
    assert math.isnan(tr["delta_g"][0])


def test_signal_kernel_rejects_nan_without_mutation():
    sig = K.DeviceSignal(DEV, 0.5, 1)
    x = torch.tensor([4.0], dtype=torch.float64, device=DEV)
    K.signal_step(sig, x, 0.1)
    before = sig.read_state()
    x.fill_(float("nan"))
    K.signal_step(sig, x, 0.1)
    after = sig.read_state()
    assert int(sig.word.item()) == N.SS_FLAG_ERR_NAN
    assert after["step_count"] == before["step_count"] == 1
    assert after["ewma_current"] == before["ewma_current"] == 4.0
    assert after["error"] == N.SS_FLAG_ERR_NAN


@pytest.mark.parametrize("n,offset", [(0, 0), (1, 0), (7, 1), (1002, 0), (1002, 2), (1 << 20, 3), (5_000_003, 0)])
def test_sgd_update_plain_matches_sgd_step(n, offset):
    w, g = rand32(n, 1), rand32(n, 2)
    wd = dev_view(w, offset)
    K.sgd_update_(wd, dev_view(g, offset), None, lr=0.1)
    want = O.sgd_step(w.astype(np.float64), g.astype(np.float64), 0.1)
    np.testing.assert_allclose(wd.double().cpu().numpy(), want, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("mu,wd,nest,damp", [(0.9, 0.0, False, 0.0), (0.9, 4e-4, False, 0.0),
                                              (0.9, 4e-4, True, 0.0), (0.5, 1e-3, False, 0.1),
                                              (0.0, 5e-4, False, 0.0)])
def test_sgd_momentum_matches_torch_rule(mu, wd, nest, damp):
    n = 100_003
    w = rand32(n, 3)
    wdev = torch.from_numpy(w).to(DEV)
    mdev = torch.zeros_like(wdev)
    w64, buf = w.astype(np.float64), None
    for k in range(6):
        g = rand32(n, 10 + k)
        K.sgd_update_(wdev, torch.from_numpy(g).to(DEV), mdev, lr=0.05, momentum=mu, dampening=damp,
                      weight_decay=wd, nesterov=nest, first_step=(k == 0))
        w64, buf = O.sgd_momentum_step(w64, g.astype(np.float64), buf, 0.05, mu, damp, wd, nest, first=(k == 0))
    np.testing.assert_allclose(wdev.double().cpu().numpy(), w64, rtol=1e-5, atol=1e-6)


def test_prescale_epilogue_reads_device_word():
    n = 4099
    w, g = rand32(n, 5), rand32(n, 6)
    word = torch.tensor([1], dtype=torch.int32, device=DEV)
    a = torch.from_numpy(w).to(DEV)
    K.sgd_update_(a, torch.from_numpy(g).to(DEV), lr=0.1, sync_word=word, sync_scale=0.25)
    b = torch.from_numpy(w).to(DEV)
    word.zero_()
    K.sgd_update_(b, torch.from_numpy(g).to(DEV), lr=0.1, sync_word=word, sync_scale=0.25)
    # power-of-two scale: exact
    assert torch.equal(a, b * 0.25)


@pytest.mark.parametrize("mom", [0.0, 0.9])
def test_fused_update_norm_equals_separate_kernels(mom):
    n = 2_000_001
    w, g = rand32(n, 7), rand32(n, 8)
    w1, w2 = torch.from_numpy(w).to(DEV), torch.from_numpy(w).to(DEV)
    m1, m2 = torch.zeros_like(w1), torch.zeros_like(w1)
    gd = torch.from_numpy(g).to(DEV)
    sig = K.DeviceSignal(DEV, 0.5, 1)
    ws = K.Workspace(DEV)
    K.update_norm_signal_(w1, gd, m1, sig, ws, lr=0.01, delta=0.1, momentum=mom, weight_decay=1e-4,
                          first_step=True)
    K.sgd_update_(w2, gd, m2, lr=0.01, momentum=mom, weight_decay=1e-4, first_step=True)
    assert torch.equal(w1, w2)  # same per-element arithmetic
    if mom:
        assert torch.equal(m1, m2)
    st = sig.read_state()
    assert st["last_norm_sq"] == pytest.approx(O.norm_sq(g.astype(np.float64)), rel=1e-12)
    assert int(sig.word.item()) == 1  # warmup step syncs


def test_replica_mean_and_flag_max():
    n = 10_007
    hosts = [rand32(n, 20 + r) for r in range(4)]
    bufs = [torch.from_numpy(h).to(DEV) for h in hosts]
    out = K.mean(bufs)
    want = O.aggregate_mean([h.astype(np.float64) for h in hosts])
    np.testing.assert_allclose(out.double().cpu().numpy(), want, rtol=1e-6, atol=1e-7)
    K.replica_average_(bufs)
    for b in bufs:
        assert torch.equal(b, out)
    words = [torch.tensor([v], dtype=torch.int32, device=DEV) for v in (0, 1, 0, 0)]
    K.replica_flag_max_(words)
    assert [int(w.item()) for w in words] == [1, 1, 1, 1]


def test_cpu_tensors_rejected_loudly():
    with pytest.raises(ConfigError):
        K.norm_sq(torch.zeros(4))
    with pytest.raises(ConfigError):
        K.sgd_update_(torch.zeros(4), torch.zeros(4), lr=0.1)


@pytest.mark.parametrize("P", [100_000_000])
def test_full_size_properties(P):
    """North-star size (100M fp32): size-independent properties."""
    gen = torch.Generator(device=DEV).manual_seed(0)
    g = torch.randn(P, generator=gen, device=DEV)
    w = torch.randn(P, generator=gen, device=DEV)
    n1 = K.norm_sq(g).item()
    assert K.norm_sq(g * 2).item() == 4 * n1
    half = P // 2 + 3
    parts = K.norm_sq_multi([g[:half], g[half:]]).item()
    assert parts == pytest.approx(n1, rel=1e-12)
    ref_torch = torch.dot(g.double(), g.double()).item()
    assert n1 == pytest.approx(ref_torch, rel=1e-11)
    # K13 with lr = 0 is the identity on w and reproduces K1's norm
    w0 = w.clone()
    sig = K.DeviceSignal(DEV, 0.08, 1)
    ws = K.Workspace(DEV)
    K.update_norm_signal_(w, g, None, sig, ws, lr=0.0, delta=0.1)
    assert torch.equal(w, w0)
    assert sig.read_state()["last_norm_sq"] == pytest.approx(n1, rel=1e-12)
    # plain update on a sampled index set vs float64
    K.sgd_update_(w, g, None, lr=0.125)
    idx = torch.randint(0, P, (100_000,), generator=gen, device=DEV)
    want = w0[idx].double() - 0.125 * g[idx].double()
    torch.testing.assert_close(w[idx].double(), want, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("offset,mom,nest,n", [(0, 0.9, 0, 300_007), (1, 0.9, 0, 300_007), (3, 0.0, 0, 65_541),
                                               (0, 0.9, 1, 1_002), (2, 0.9, 0, 1_000_003)])
def test_step_plan_is_bit_identical_to_the_per_call_entry_point(offset, mom, nest, n):
    """ss_step_plan_init/launch (the per-step path of SelSyncStep) and
    ss_update_norm_signal_f32 (every argument per call) on the same inputs:
    the same parameters, momentum, votes and trace rows, bit for bit --
    misaligned heads, the one-block grid (n = 1,002) and ragged tails included."""
    import ctypes

    lr, wd, delta = 0.05, 4e-4, 0.2  # the step-4 Delta (0.07) is local, the rest sync
    w0 = rand32(n, 1, 0.1)
    grads = [dev_view(rand32(n, 10 + s, 1.0 + 0.3 * (s % 3)), offset) for s in range(7)]
    runs = []
    for use_plan in (False, True):
        w = dev_view(w0, offset)
        m = dev_view(np.zeros(n, np.float32), offset)
        sig = K.DeviceSignal(DEV, 0.5, 2, 64)
        ws = K.Workspace(DEV)
        stream = torch.cuda.current_stream().cuda_stream
        if use_plan:
            desc = N.RankStepC(w.data_ptr(), grads[0].data_ptr(), m.data_ptr() if mom else None, n, mom, 0.0, wd,
                               nest, sig.state.data_ptr(), delta, sig.word.data_ptr(), sig.trace.data_ptr(), 64, 0,
                               None, ws.ptr)
            plan = N.StepPlanC()
            N.check(N.LIB.ss_step_plan_init(ctypes.addressof(plan), ctypes.addressof(desc), 0))
        words = []
        for s, g in enumerate(grads):
            if use_plan:
                N.check(N.LIB.ss_step_plan_launch(ctypes.addressof(plan), g.data_ptr(), lr, int(s == 0), stream))
            else:
                K.update_norm_signal_(w, g, m if mom else None, sig, ws, lr=lr, delta=delta, momentum=mom,
                                      weight_decay=wd, nesterov=bool(nest), first_step=s == 0)
            words.append(int(sig.word.item()))
        torch.cuda.synchronize()
        runs.append((w.cpu().numpy().copy(), m.cpu().numpy().copy(), words, sig.read_trace()[:7].tobytes()))
    (wa, ma, da, ta), (wb, mb, db, tb) = runs
    assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
    assert np.array_equal(ma.view(np.uint32), mb.view(np.uint32))
    assert da == db and 0 < sum(x & 1 for x in da) < len(da)
    assert ta == tb
