# compute-sanitizer racecheck / synccheck / memcheck on the production decode
# kernels at small n (tools/sanitize_decode.py); summaries -> gpurun_out/san_*.txt
mkdir -p gpurun_out
N=${1:-15}
for tool in memcheck synccheck racecheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 python tools/sanitize_decode.py $N > gpurun_out/san_$tool.txt 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_$tool.txt | tail -2 | tr '\n' ' ')"
done
