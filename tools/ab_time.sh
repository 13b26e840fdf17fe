#!/bin/bash
# Same-box A/B timing of library variants: tools/ab_time.sh "<command>" _ab/A.so _ab/B.so ...
# Each variant is copied over the in-tree library and the command run, twice
# round-robin (box clocks drift between boxes; compare within one call).
cmd="$1"; shift
lib=paper_2512_02371_b200/_native/libtsb200.so
cp "$lib" /tmp/ab_orig.so
for round in 1 2; do
  for v in "$@"; do
    cp "$v" "$lib"
    echo "== $v: $(eval "$cmd" 2>&1 | tail -1)"
  done
done
cp /tmp/ab_orig.so "$lib"
