"""The C-ABI library loads on a CPU-only machine and exports exactly what
include/selsync_b200.h declares; host entry points work without a GPU."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "selsync_b200.h").read_text()
    return sorted(set(re.findall(r"SS_API\s+(?:const\s+)?\w+\*?\s+\**(ss_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert len(syms) >= 20
    for must in ("ss_norm_sq_f32", "ss_update_norm_signal_f32", "ss_signal_step",
                 "ss_sgd_update_f32", "ss_signal_observe", "ss_decide"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2307_07950_b200 import _native as N

    lib = ctypes.CDLL(str(N.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding covers every declared symbol
    assert sorted(N.EXPORTED) == declared_symbols()


def test_struct_layouts():
    from paper_2307_07950_b200 import _native as N

    assert N.LIB.ss_signal_state_size() == ctypes.sizeof(N.SignalStateC) == 64
    assert N.LIB.ss_trace_row_size() == ctypes.sizeof(N.TraceRowC) == 32
    assert N.LIB.ss_abi_version() == 1
    assert N.workspace_bytes() > 8 * 148


def test_symm_group_layout_matches_ctypes_mirror():
    """Every field offset of ss_symm_group (and its size) as compiled into the
    library equals the ctypes mirror the package passes to the step kernels."""
    from paper_2307_07950_b200 import _native as N

    cap = 64
    offs = (ctypes.c_int64 * cap)()
    count = ctypes.c_int32(0)
    N.check(N.LIB.ss_symm_group_layout(offs, cap, ctypes.byref(count)))
    names = [f[0] for f in N.SymmGroupC._fields_]
    assert count.value == len(names) + 1
    want = [getattr(N.SymmGroupC, n).offset for n in names] + [ctypes.sizeof(N.SymmGroupC)]
    assert list(offs[: count.value]) == want
    with pytest.raises(N.ConfigError):
        N.check(N.LIB.ss_symm_group_layout(offs, 3, ctypes.byref(count)))


def test_error_codes_map_to_reference_exceptions():
    from paper_2307_07950_b200 import _native as N
    from paper_2307_07950_b200.errors import ConfigError, SignalError

    with pytest.raises(SignalError):
        N.check(N.LIB.ss_check_delta(-1.0))
    out = ctypes.c_double()
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_default_smoothing(0, ctypes.byref(out)))
    # device entry points validate arguments before touching the GPU
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_norm_sq_f32(None, 10, None, None, None))
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_sgd_update_f32(None, None, None, -1, 0.1, 0, 0, 0, 0, 0, None, 1.0, None))
    # the known-sync predicate validates like decide (DeltaThreshold rules)
    st = N.SignalStateC()
    st.smoothing, st.warmup = 0.5, 3
    known = ctypes.c_int32(-1)
    with pytest.raises(SignalError):
        N.check(N.LIB.ss_sync_known_ahead(ctypes.byref(st), float("nan"), ctypes.byref(known)))
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_sync_known_ahead(None, 0.1, ctypes.byref(known)))
    N.check(N.LIB.ss_sync_known_ahead(ctypes.byref(st), 0.1, ctypes.byref(known)))
    assert known.value == 1  # step_count 0 < warmup
    # the one-launch step rejects a missing group before any launch
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_step_symm_f32(None, None, None, 0, 0.1, 0, 0, 0, 0, 0, ctypes.byref(st), 0.1,
                                       None, None, 0, None, None, None))


def test_rank_step_layout_matches_ctypes_mirror():
    """ss_rank_step's compiled field offsets and size, and the size of the
    opaque ss_step_plan, equal the ctypes mirrors the package builds plans from."""
    from paper_2307_07950_b200 import _native as N

    offs = (ctypes.c_int64 * 32)()
    count = ctypes.c_int32(0)
    N.check(N.LIB.ss_rank_step_layout(offs, 32, ctypes.byref(count)))
    names = [f[0] for f in N.RankStepC._fields_]
    want = [getattr(N.RankStepC, n).offset for n in names] + [ctypes.sizeof(N.RankStepC),
                                                              ctypes.sizeof(N.StepPlanC)]
    assert list(offs[: count.value]) == want


def test_step_plan_validates_before_any_launch():
    """ss_step_plan_init checks what the per-call entry points check; a plan
    that was never (successfully) initialised refuses to launch."""
    from paper_2307_07950_b200 import _native as N
    from paper_2307_07950_b200.errors import ConfigError, SignalError

    plan = N.StepPlanC()
    with pytest.raises(ConfigError, match="not initialised"):
        N.check(N.LIB.ss_step_plan_launch(ctypes.addressof(plan), 16, 0.1, 0, None))
    with pytest.raises(ConfigError):
        N.check(N.LIB.ss_step_plan_init(None, None, 0))
    st = N.SignalStateC()
    desc = N.RankStepC(16, 32, 48, 100, 0.9, 0.0, 4e-4, 0, ctypes.addressof(st), 0.3, 64, None, 0, 0, None, 80)
    cases = [
        (dict(momentum=-1.0), ConfigError),            # make_sgd_args
        (dict(nesterov=1, dampening=0.5), ConfigError),
        (dict(m=None), ConfigError),                   # momentum buffer required
        (dict(delta=-0.5), SignalError),               # DeltaThreshold
        (dict(trace=96, trace_cap=0), ConfigError),
        (dict(ws=None), ConfigError),
    ]
    for change, exc in cases:
        d = N.RankStepC.from_buffer_copy(desc)
        for k, v in change.items():
            setattr(d, k, v)
        with pytest.raises(exc):
            N.check(N.LIB.ss_step_plan_init(ctypes.addressof(plan), ctypes.addressof(d), 0))
        with pytest.raises(ConfigError, match="not initialised"):  # a failed init leaves no plan
            N.check(N.LIB.ss_step_plan_launch(ctypes.addressof(plan), 16, 0.1, 0, None))
    # gradient aggregation needs a symmetric group
    with pytest.raises(ConfigError, match="symmetric group"):
        N.check(N.LIB.ss_step_plan_init(ctypes.addressof(plan), ctypes.addressof(desc), 1))


def test_build_flags_target_sm100a():
    from paper_2307_07950_b200 import _build

    assert "arch=compute_100a,code=sm_100a" in _build.ARCH
    assert "-lineinfo" in _build.FLAGS
