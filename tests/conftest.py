"""Shared pytest wiring.

Markers: ``gpu`` = needs a CUDA device (run on a B200 via gpurun); everything
else runs on the CPU build container. The repo root is put on sys.path so the
tests import the package, the oracle (as the checker only) and the golden
fixtures the same way on both machines.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def _load_cases():
    z = np.load(GOLDEN / "selsync_cases.npz")
    meta = json.loads(bytes(z["meta_json"]).decode())
    cases = {}
    for name, m in meta.items():
        c = dict(m)
        for k in ("init", "grad_norm_sq", "ewma", "delta_g", "decision", "finals",
                  "snap_steps", "snaps"):
            c[k] = z[f"{name}/{k}"]
        cases[name] = c
    return cases


@pytest.fixture(scope="session")
def golden_cases():
    return _load_cases()


@pytest.fixture(scope="session")
def seldp_golden():
    return dict(np.load(GOLDEN / "seldp_cases.npz"))


def case_names():
    z = np.load(GOLDEN / "selsync_cases.npz")
    return sorted(json.loads(bytes(z["meta_json"]).decode()))
