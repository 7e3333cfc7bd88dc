"""Summarise ncu output for profiles/: a --set full report (.ncu-rep) and/or a
launch-list CSV (gpu__time_duration.sum per launch).

python tools/ncu_summary.py --rep gpurun_out/prof_k13.ncu-rep --launches gpurun_out/launches.csv \
    --out profiles/r01_k13 [--P 100000000 --alg-bytes 2000000000]
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_drain_per_warp_active.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def rep_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": r[i], "unit": units[i]}
        res.append(d)
    return res


def to_si(ent):
    v = float(ent["value"].replace(",", ""))
    return v * SCALE.get(ent["unit"], 1)


def launches(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"][:110]
        t = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1e-9)
        agg[name][0] += 1
        agg[name][1] += t
        order.append((name, t))
    return agg, order


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--P", type=int)
    ap.add_argument("--alg-bytes", type=float)
    a = ap.parse_args()
    summary = {}
    md = []
    if a.rep:
        rows = rep_rows(a.rep)
        summary["full"] = rows
        md.append(f"## ncu --set full: {a.rep}\n")
        for r in rows:
            md.append(f"### {r['kernel'][:120]}\n")
            for k in KEYS:
                if k in r:
                    md.append(f"- {k}: {r[k]['value']} {r[k]['unit']}")
            t = to_si(r["gpu__time_duration.sum"])
            rd, wr = to_si(r["dram__bytes_read.sum"]), to_si(r["dram__bytes_write.sum"])
            md.append(f"- derived: dram traffic {(rd + wr) / 1e9:.3f} GB/launch, "
                      f"{(rd + wr) / t / 1e9:.0f} GB/s under ncu (cold, serialised)")
            if a.alg_bytes:
                md.append(f"- algorithmic bytes {a.alg_bytes / 1e9:.3f} GB -> traffic/algorithmic = "
                          f"{(rd + wr) / a.alg_bytes:.3f}; algorithmic GB/s under ncu {a.alg_bytes / t / 1e9:.0f}")
            md.append("")
        if a.P and rows:
            r = rows[-1]
            summary["traffic"] = {str(a.P): {
                "dram_bytes_per_launch": to_si(r["dram__bytes_read.sum"]) + to_si(r["dram__bytes_write.sum"]),
                "kernel": r["kernel"], "source": a.rep}}
    if a.launches:
        agg, order = launches(a.launches)
        total = sum(v[1] for v in agg.values())
        md.append(f"## launch list: {a.launches} ({len(order)} launches, {total * 1e3:.3f} ms total)\n")
        md.append("| kernel | launches | total ms | share |")
        md.append("|---|---|---|---|")
        for name, (cnt, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| `{name}` | {cnt} | {t * 1e3:.3f} | {t / total:.1%} |")
        summary["launches"] = {k: {"count": v[0], "total_s": v[1]} for k, v in agg.items()}
    with open(a.out + ".md", "w") as fh:
        fh.write("\n".join(md) + "\n")
    with open(a.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
