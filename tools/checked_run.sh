# The checked build (tools/checked_build.sh) on the production launch shapes:
# bounds asserts + NaN-poisoned shared memory + per-warp schedule jitter, every
# result compared with the oracle; -> gpurun_out/checked_*.log
export PQ_LIB_PATH=variants/checked.so
mkdir -p gpurun_out
for n in 12 15 16; do
  timeout 900 python tools/sanitize_decode.py $n > gpurun_out/checked_decode_n$n.log 2>&1; echo "shapes n=$n rc=$? $(grep -c ok gpurun_out/checked_decode_n$n.log) ok, $(grep -c MISMATCH gpurun_out/checked_decode_n$n.log) mismatches"
done
timeout 2400 python -m pytest tests/test_bench_shapes.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "bench or sweep or repeat or cluster or wide or fixed or config_parity" > gpurun_out/checked_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/checked_tests.log
