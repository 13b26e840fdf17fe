#!/bin/bash
# axis-pass knob sweep (same box): tools/sweep_apass.sh "NBGS" "RINGS" GEOMETRIES...
#   e.g. tools/sweep_apass.sh "- 2 4" "- 3 4 6" 921 540    ("-" = default)
nbgs="$1"; rings="$2"; shift 2
for nbg in $nbgs; do
  for ring in $rings; do
    env=""
    [ "$nbg" != "-" ] && env="$env TSB_APASS_NBG=$nbg"
    [ "$ring" != "-" ] && env="$env TSB_APASS_RING=$ring"
    echo "nbg=$nbg ring=$ring: $(env $env python tools/time_apass.py "$@" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['cfg'], 'v', d['v_ms'], 'h', d['h_ms'], end=' | ')")"
  done
done
