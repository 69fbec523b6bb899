# parity of a variant .so on the bench shapes (bench.py's own oracle check of every timed frame)
# VARIANTS="a" CFGS="c3 c5" bash tools/ab_parity.sh
VARIANTS=${VARIANTS:-"v0"}; CFGS=${CFGS:-"c3"}
for c in $CFGS; do for v in $VARIANTS; do
  r=$(PQ_LIB_PATH=variants/$v.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-extras --steps 3 2>&1 | tail -1)
  echo "$c $v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d.get("parity"))' 2>&1 | tail -1)"
done; done
