# A/B: bench c3 for each variant .so (variants/<v>.so) and f mode given
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-"v0 vC vD"}; MODES=${MODES:-"fixed fast"}; CFG=${CFG:-c3}
for v in $VARIANTS; do for m in $MODES; do
  r=$(PQ_LIB_PATH=variants/$v.so timeout 200 python bench.py --config $CFG --fmode $m --no-cpu-baseline --steps 5 2>&1 | tail -1)
  echo "$v $m $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"].get("band_share"), d["roofline"].get("upper_band"))' 2>&1 | tail -1)"
done; done
