#!/bin/bash
# bench frac of several configs (one line): tools/ab_cfgs.sh
out=""
for c in c2 c3-9 c3-31 c5; do
  v=$(python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['frac'])")
  out="$out $c=$v"
done
for f in 24 32; do
  v=$(python bench.py --frames $f --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['frac'])")
  out="$out c2x$f=$v"
done
echo $out
