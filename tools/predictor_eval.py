"""Replay the step-order choice of the one-launch step on decision traces and
price it with the measured per-order step costs (P = 100M).

Traces: the agreed decisions of the reference's golden runs
(tests/golden/selsync_cases.npz, produced by the unmodified reference) and the
bench's alternating mix. Order rules, as the kernel implements them
(csrc/selsync_step.cu): a single EWMA of the agreed decisions (weight 1/4,
this round's first version), the 2-bit-history predictor (an EWMA per context
of the previous two decisions), always update-first, always norm-first, and a
perfect oracle. Steps whose decision is known ahead (warmup, delta == 0) take
the known-sync pass whatever the rule. Prints ms/step per trace and rule.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
# ms per step at P = 100M (profiles/r01_predictor, r01_known_sync)
COST = {2: dict(uf_local=0.337, nf_local=0.394, uf_sync=0.956, nf_sync=0.715, known=0.660),
        4: dict(uf_local=0.342, nf_local=0.397, uf_sync=1.260, nf_sync=1.020, known=0.961)}
THRESHOLD = 0.2


def rule_ewma():
    p = [0.0]

    def pick(_t):
        return p[0] >= THRESHOLD

    def update(s):
        p[0] = 0.75 * p[0] + (0.25 if s else 0.0)
    return pick, update


def rule_2bit():
    pr = [0.0] * 4
    h = [0]

    def pick(_t):
        return pr[h[0]] >= THRESHOLD

    def update(s):
        pr[h[0]] = 0.75 * pr[h[0]] + (0.25 if s else 0.0)
        h[0] = ((h[0] << 1) | int(s)) & 3
    return pick, update


def price(trace, known, n, rule):
    c = COST[n]
    total = 0.0
    if rule in ("ewma", "2bit"):
        pick, update = (rule_ewma if rule == "ewma" else rule_2bit)()
    for t, s in enumerate(trace):
        if rule in ("ewma", "2bit", "oracle") and known[t]:
            total += c["known"]
        elif rule == "oracle":
            total += c["nf_sync"] if s else c["uf_local"]
        else:
            nf = {"uf": False, "nf": True}.get(rule)
            if nf is None:
                nf = pick(t)
            total += c[("nf_" if nf else "uf_") + ("sync" if s else "local")]
        if rule in ("ewma", "2bit"):
            update(s)
    return total / len(trace)


def main():
    z = np.load(ROOT / "tests" / "golden" / "selsync_cases.npz")
    meta = json.loads(bytes(z["meta_json"]).decode())
    traces = []
    for name, m in meta.items():
        if m["aggregation"] != "params":
            continue
        d = z[f"{name}/decision"]
        d = d.any(axis=1) if d.ndim > 1 else d
        known = [t < m["warmup"] or m["delta"] == 0.0 for t in range(len(d))]
        traces.append((name, list(map(bool, d)), known))
    alt = [bool(k % 2) for k in range(200)]
    traces.append(("bench mix (L,S alternating, warmup 1)", alt, [k == 0 for k in range(200)]))
    rules = ["uf", "nf", "ewma", "2bit", "oracle"]
    for n in (2, 4):
        print(f"N = {n}: ms/step at P = 100M (known-sync pass on warmup / delta = 0 steps for the adaptive rules)")
        print(f"  {'trace':40s} " + " ".join(f"{r:>7s}" for r in rules))
        for name, d, known in traces:
            row = [price(d, known, n, r) for r in rules]
            print(f"  {name:40s} " + " ".join(f"{v:7.3f}" for v in row))
    return 0


if __name__ == "__main__":
    sys.exit(main())
