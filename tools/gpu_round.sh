timeout 1200 python -m pytest tests/test_bench_shapes.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fixed or q88 or bench or sweep or repeat or cluster or wide or pipelined or trials" > gpurun_out/c3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c3_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/c3_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/c3_bench.log | cut -c1-600
for c in c4 c5 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c3_bench_$c.log 2>&1; tail -1 gpurun_out/c3_bench_$c.log | cut -c1-300; done
