# source-level ncu capture of the upper band in isolation (tools/upper_only.py, 256 frames)
# usage: bash tools/upper_src.sh <variant.so> <tag>
V=${1:-variants/base.so}; TAG=${2:-upper}
mkdir -p gpurun_out
PQ_LIB_PATH=$V timeout 900 ncu --set full --clock-control none --import-source on -k regex:sc_decode -s 3 -c 1 \
    -o gpurun_out/src_${TAG} -f python tools/upper_only.py 256 fixed > gpurun_out/src_${TAG}_run.log 2>&1
echo "capture rc=$?"
ncu -i gpurun_out/src_${TAG}.ncu-rep --page raw --csv > gpurun_out/src_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/src_${TAG}.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/src_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_sass.csv 2>/dev/null
ls -la gpurun_out/src_${TAG}*
