#!/bin/bash
# EXTRA="-D..." census_build.sh <name>: compile polarsc.cu alone (fixed-point kernels) to a cubin and print,
# per production kernel, the indicators of the serial engine's compiled form: body / w32 / walk instruction
# counts, R2UR in w32 (0 = the fast form), STL in walk and in w32 (0 = no spills).  CPU only, ~2.5 min.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/census_$1; mkdir -p $T
nvcc -w -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -ftz=false -DPQ_ONLY_FIXED $EXTRA \
     -I "$ROOT/include" -cubin -o $T/k.cubin "$ROOT/paper_1204_5882_b200/csrc/polarsc.cu"
nvdisasm -c $T/k.cubin > $T/all.dis 2>/dev/null
for K in ILi3ELb0ELb0ELi256ELi0E ILi3ELb1ELb0ELi512ELi4E ILi3ELb1ELb0ELi512ELi0E; do
  awk -v K=$K '
    /^\$?_Z[^ ]*:$/ { cur=$1; next }
    /^ +\/\*[0-9a-f]+\*\// { if (index(cur,K)==0) next;
        f = (index(cur,"_ZN2se3w32Eij")>0) ? "w32" : (index(cur,"_ZN2se4walk")>0) ? "walk" : (index(cur,"$")==0 || index(cur,"$")==1 && index(substr(cur,2),"$")==0) ? "body" : "other";
        n[f]++; if ($0 ~ /R2UR/) r[f]++; if ($0 ~ / STL/) s[f]++; }
    END { printf "%s body=%d w32=%d walk=%d | w32.R2UR=%d w32.STL=%d walk.STL=%d body.STL=%d\n", K, n["body"], n["w32"], n["walk"], r["w32"], s["w32"], s["walk"], s["body"] }' $T/all.dis
done
