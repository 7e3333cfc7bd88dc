"""Build the sm_100a shared library in-tree with nvcc (no JIT cache).

``python -m paper_2307_07950_b200._build`` or ``__graft_entry__.build()``.
The library lands at ``paper_2307_07950_b200/_lib/libselsync_b200.so`` so it
travels to the GPU box inside the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRCS = [PKG / "csrc" / f for f in ("selsync_b200.cu", "selsync_symm.cu", "selsync_step.cu", "selsync_multi.cu")]
DEPS = [*SRCS, *sorted((PKG / "csrc").glob("*.cuh"))]
HEADER = ROOT / "include" / "selsync_b200.h"
OUT = PKG / "_lib" / "libselsync_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-shared",
    "-Xcompiler",
    "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-Xptxas",
    "-v",
    "--expt-relaxed-constexpr",
]
LIBS: list[str] = []


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libselsync_b200.so")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    mtime = OUT.stat().st_mtime
    return any(p.stat().st_mtime > mtime for p in (*DEPS, HEADER))


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, *FLAGS, f"-I{HEADER.parent}", *map(str, SRCS), *LIBS, "-o", str(tmp)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (OUT.parent / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed ({proc.returncode}):\n{log[-4000:]}")
    if "spill" in log and verbose:
        print(log, file=sys.stderr)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose=True)
    print(path)
