# A/B: bench each variant .so (variants/<v>.so) on the configs given, fixed point
# VARIANTS="a b" CFGS="c3 c4" bash tools/ab_run.sh
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-"v0"}; CFGS=${CFGS:-"c3"}; STEPS=${STEPS:-10}
for c in $CFGS; do for v in $VARIANTS; do
  r=$(PQ_LIB_PATH=variants/$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-parity --no-extras --steps $STEPS 2>&1 | tail -1)
  echo "$c $v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["kernel_ms"], d.get("band_share"))' 2>&1 | tail -1)"
done; done
