# Copy one profile round's outputs (tools/profile_round.sh <cfg> fixed <tag> + bench logs)
# into profiles/r01: bash tools/save_profiles.sh <tag> <bench-suffix>
TAG=$1; SUF=$2; P=${P:-profiles/r01}
python tools/launch_summary.py gpurun_out/prof_${TAG}_launches.csv "python bench.py --config c3 --fmode fixed --steps 2 --warmup 3 --no-cpu-baseline" > $P/ncu_launches_c3_fixed_summary.txt
cp gpurun_out/prof_${TAG}_launches.csv $P/ncu_launches_c3_fixed.csv
python tools/ncu_summary.py gpurun_out/prof_${TAG}_full_raw.csv c3 fixed $P/ncu_full_c3_fixed.json > /dev/null
tail -1 gpurun_out/prof_${TAG}_bench.log > $P/bench_c3_fixed.json
for c in c2 c4 c5; do [ -f gpurun_out/bench_${c}_${SUF}.log ] && tail -1 gpurun_out/bench_${c}_${SUF}.log > $P/bench_${c}_fixed.json; done
for c in c3 c5; do [ -f gpurun_out/bench_${c}_exact_${SUF}.log ] && tail -1 gpurun_out/bench_${c}_exact_${SUF}.log > $P/bench_${c}_exact.json; done
P=$P python - "$TAG" <<'PY'
import csv, sys
rows = list(csv.reader(open(f'gpurun_out/prof_{sys.argv[1]}_full_details.csv')))
want = {'DRAM Throughput', 'Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'Executed Ipc Active',
        'Issue Slots Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Registers Per Thread', 'Dynamic Shared Memory Per Block', 'Achieved Occupancy'}
h = rows[0]; ci = {c: i for i, c in enumerate(h)}
out = ['ncu --set full, sc_decode_kernel<3> (fixed point), c3, 256 frames (tools/profile_round.sh)']
seen = set()
for r in rows[1:]:
    if len(r) > ci['Metric Value'] and r[ci['Metric Name']] in want:
        k = (r[ci['Section Name']], r[ci['Metric Name']])
        if k not in seen:
            seen.add(k)
            out.append(f"{k[0]:35s} {k[1]:40s} {r[ci['Metric Value']]:>12s} {r[ci['Metric Unit']]}")
open('' + __import__("os").environ.get("P", "profiles/r01") + '/ncu_full_c3_fixed_details.txt', 'w').write('\n'.join(out) + '\n')
PY
