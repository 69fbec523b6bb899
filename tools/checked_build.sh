# PQ_CHECKED library (bounds asserts, poisoned shared memory, schedule jitter)
# -> variants/checked.so, all f modes; [EXTRA="-D..."] checked_build.sh [name]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/variants"
nvcc -w -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -ftz=false -DPQ_CHECKED $EXTRA -I "$ROOT/include" \
     -Xcompiler -fPIC -shared -cudart static -o "$ROOT/variants/${1:-checked}.so" "$ROOT/paper_1204_5882_b200/csrc/polarsc.cu" "$ROOT/paper_1204_5882_b200/csrc/verify.cu" "$ROOT/paper_1204_5882_b200/csrc/de.cu" "$ROOT/paper_1204_5882_b200/csrc/codetable.cu" "$ROOT/paper_1204_5882_b200/csrc/frames.cu"
