"""Where do the step kernels touch local memory? Compiles one translation unit
to a cubin with -lineinfo and lists, per kernel, the source lines of every
STL/LDL (spill store / load) instruction, so a spill reported by ptxas -v can
be checked against the hot loops (sgd_pass / sgd_block_range / the means).

    python tools/spill_sites.py [paper_2307_07950_b200/csrc/selsync_step.cu] [kernel-substring]
"""

import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    src = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2307_07950_b200/csrc/selsync_step.cu"
    pick = sys.argv[2] if len(sys.argv) > 2 else ""
    with tempfile.TemporaryDirectory() as tmp:
        cubin = Path(tmp) / "k.cubin"
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                        f"-I{ROOT / 'include'}", "-cubin", "-o", str(cubin), str(src)], check=True)
        sass = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True, text=True).stdout
    fn, cur, sites = None, None, {}
    for line in sass.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", line)
        if m:
            fn = m.group(1)
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{Path(m.group(1)).name}:{m.group(2)}"
        if fn and pick in fn and re.search(r"\b(STL|LDL)", line):
            sites.setdefault(fn, {}).setdefault(cur, 0)
            sites[fn][cur] += 1
    for fn, s in sites.items():
        name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        print(name.replace("(anonymous namespace)::", "").split("(")[0])
        for where, k in sorted(s.items(), key=lambda kv: kv[0] or ""):
            print(f"    {k:3d} x  {where}")


if __name__ == "__main__":
    main()
