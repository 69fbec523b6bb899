#!/bin/bash
# [EXTRA="-D..."] build_variant.sh <name>: compile a fixed-point-only libpolarsc.so
# (-DPQ_ONLY_FIXED, same flags as build.py plus $EXTRA) into variants/<name>.so for
# A/B runs via PQ_LIB_PATH (tools/ab_run.sh).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/variants"
nvcc -w -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -ftz=false -DPQ_ONLY_FIXED $EXTRA -I "$ROOT/include" \
     -Xcompiler -fPIC -shared -cudart static -o "$ROOT/variants/$1.so" "$ROOT/paper_1204_5882_b200/csrc/polarsc.cu" "$ROOT/paper_1204_5882_b200/csrc/verify.cu" "$ROOT/paper_1204_5882_b200/csrc/de.cu" "$ROOT/paper_1204_5882_b200/csrc/codetable.cu" "$ROOT/paper_1204_5882_b200/csrc/frames.cu"
