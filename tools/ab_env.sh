#!/bin/bash
# Same-box A/B of environment settings: tools/ab_env.sh "<command>" "ENV_A" "ENV_B" ...
# ("-" = no extra environment); three rounds, round-robin.
cmd="$1"; shift
for round in 1 2 3; do
  for e in "$@"; do
    if [ "$e" = "-" ]; then out=$(eval "$cmd" 2>&1 | tail -1); else out=$(env $e bash -c "$cmd" 2>&1 | tail -1); fi
    echo "== [$e] $out"
  done
done
