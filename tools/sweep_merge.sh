#!/bin/bash
# fused-kernel super-block merge threshold sweep (same box): tools/sweep_merge.sh
for c in c3-21 c3-31 c5 c2; do
  for env in "TSB_MERGE_GAIN=0.0" "TSB_MERGE_GAIN=0.05" "TSB_MERGE_GAIN=0.15" "TSB_NO_MERGE=1"; do
    r=$(env $env python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])")
    echo "$c $env $r"
  done
done
