# Profile the default bench config on one GPU (run under gpurun):
#   1. bench.py without any profiler (the number), 2. the ncu launch list of
#   the same command, 3. one `ncu --set full` capture of sc_decode_kernel,
#   exported as raw CSV.  Outputs: gpurun_out/prof_<tag>_*.
# usage: bash tools/profile_round.sh <config> <fmode> <tag>
CFG=${1:-c3}; FM=${2:-fixed}; TAG=${3:-$CFG}
mkdir -p gpurun_out
timeout 300 python bench.py --config $CFG --fmode $FM > gpurun_out/prof_${TAG}_bench.log 2>&1 || exit 1
tail -1 gpurun_out/prof_${TAG}_bench.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/prof_${TAG}_launches.csv \
    python bench.py --config $CFG --fmode $FM --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof_${TAG}_launch_run.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sc_decode -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_full -f \
    python tools/prof_decode.py --config $CFG --fmode $FM > gpurun_out/prof_${TAG}_full_run.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/prof_${TAG}_full.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_full_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}_full.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_full_details.csv 2>/dev/null
echo done
