# A/B one bench flag: bash tools/ab_flag.sh "<flag values...>" "<configs>" (flag given as e.g. "--warp-log2 8")
FLAGS=${FLAGS:-"--warp-log2 8|--warp-log2 9"}; CFGS=${CFGS:-"c3"}
IFS='|' read -ra FL <<< "$FLAGS"
for c in $CFGS; do for f in "${FL[@]}"; do
  r=$(timeout 300 python bench.py --config $c --no-cpu-baseline --steps 5 $f 2>&1 | tail -1)
  echo "$c [$f] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"].get("band_share"))' 2>&1 | tail -1)"
done; done
