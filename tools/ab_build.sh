#!/bin/bash
# Build a variant of libselsync_b200.so with extra -D flags into _lib/ab/<name>.so
# for same-box A/B timing (load it with SS_LIB_PATH=...). Usage: tools/ab_build.sh NAME -DFLAG ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p paper_2307_07950_b200/_lib/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC,-ffp-contract=off,-fvisibility=hidden \
  --expt-relaxed-constexpr -Iinclude "$@" paper_2307_07950_b200/csrc/selsync_b200.cu paper_2307_07950_b200/csrc/selsync_symm.cu \
  paper_2307_07950_b200/csrc/selsync_step.cu paper_2307_07950_b200/csrc/selsync_multi.cu -o paper_2307_07950_b200/_lib/ab/$name.so
echo built paper_2307_07950_b200/_lib/ab/$name.so
