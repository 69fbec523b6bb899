timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/c4_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c4_gputests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c4_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/c4_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print({k:d[k] for k in ('value','ms_per_step','kernel_ms','e2e','parity')})
print(d['roofline']['frac'], d['band_share'], d['clocks'])
for k,v in d.get('configs',{}).items(): print(k, v['value'], v['ms_per_step'], v['e2e']['value'] if v['e2e'] else None, v['parity']['mismatches'], v['roofline']['frac'])
"
