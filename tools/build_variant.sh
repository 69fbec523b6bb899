#!/bin/bash
# [EXTRA="-D..."] build_variant.sh <source.cu> <name>: compile an alternative libpolarsc.so into
# variants/<name>.so (same flags as build.py) for A/B runs via PQ_LIB_PATH.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
tmp="$ROOT/paper_1204_5882_b200/csrc/_variant_$2.cu"
cp "$1" "$tmp"
mkdir -p "$ROOT/variants"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -ftz=false $EXTRA -I "$ROOT/include" \
     -Xcompiler -fPIC -shared -cudart static -o "$ROOT/variants/$2.so" "$tmp" "$ROOT/paper_1204_5882_b200/csrc/verify.cu" "$ROOT/paper_1204_5882_b200/csrc/de.cu" || { rm -f "$tmp"; exit 1; }
rm -f "$tmp"
