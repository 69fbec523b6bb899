# ncu --set full capture (with source-level stall sampling) of the production
# sc_decode_kernel on a config's bench batch; exports raw / details / source
# pages under gpurun_out/src_<tag>_*.  usage: bash tools/gpu_prof_src.sh <cfg> <fmode> <tag> [frames]
CFG=${1:-c3}; FM=${2:-fixed}; TAG=${3:-$CFG}; FR=${4:-0}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sc_decode -s 1 -c 1 \
    -o gpurun_out/src_${TAG} -f \
    python tools/prof_decode.py --config $CFG --fmode $FM --frames $FR > gpurun_out/src_${TAG}_run.log 2>&1
echo "capture rc=$?"
ncu -i gpurun_out/src_${TAG}.ncu-rep --page raw --csv > gpurun_out/src_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/src_${TAG}.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/src_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/src_${TAG}.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${TAG}_cuda.csv 2>/dev/null
ls -la gpurun_out/src_${TAG}*
