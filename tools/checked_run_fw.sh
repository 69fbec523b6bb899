# The checked build with the optional ring paths compiled in for every kernel (PQ_FUSE2=1: two upper steps per
# pass; PQ_RING_WARPREL=1: per-warp stage release, 3 stages): EXTRA="-DPQ_ONLY_FIXED -DPQ_FUSE2=1
# -DPQ_RING_WARPREL=1" bash tools/checked_build.sh checked_fw; every decode compared with the oracle.
export PQ_LIB_PATH=variants/checked_fw.so PQ_FIXED_ONLY=1
mkdir -p gpurun_out
for n in 15 16; do
  timeout 900 python tools/sanitize_decode.py $n > gpurun_out/checked_fw_n$n.log 2>&1; echo "fw shapes n=$n rc=$? $(grep -c ok gpurun_out/checked_fw_n$n.log) ok, $(grep -c MISMATCH gpurun_out/checked_fw_n$n.log) mismatches"
done
PQ_SHAPES="2,256,13;4,256,13;1,256,13;1,256,14;2,0,14" timeout 900 python tools/sanitize_decode.py 17 > gpurun_out/checked_fw_n17.log 2>&1; echo "fw shapes n=17 rc=$? $(grep -c ok gpurun_out/checked_fw_n17.log) ok, $(grep -c MISMATCH gpurun_out/checked_fw_n17.log) mismatches"
PQ_SHAPES="4,0,14;2,256,13" timeout 900 python tools/sanitize_decode.py 18 > gpurun_out/checked_fw_n18.log 2>&1; echo "fw shapes n=18 rc=$? $(grep -c ok gpurun_out/checked_fw_n18.log) ok, $(grep -c MISMATCH gpurun_out/checked_fw_n18.log) mismatches"
timeout 1800 python -m pytest tests/test_bench_shapes.py -q -p no:cacheprovider -k "fixed and (bench or sweep or repeat)" > gpurun_out/checked_fw_tests.log 2>&1; echo "fw tests rc=$?"; tail -2 gpurun_out/checked_fw_tests.log
