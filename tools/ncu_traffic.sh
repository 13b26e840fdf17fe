#!/bin/bash
# ncu --set full of one pipeline call per bench config -> gpurun_out/traffic/<cfg>_<frames>.ncu-rep
mkdir -p gpurun_out/traffic
cp profiles/ncu_summary.json gpurun_out/ncu_summary_traffic.json
for c in c1 c3-9 c3-15 c3-21 c3-31 c5 c6-143 c6-245 c6-450 c6-921; do
  f=4; [ "${c%%-*}" = "c3" ] && f=1
  python tools/ncu_traffic.py run $c $f || { echo "$c failed"; continue; }
  timeout 600 ncu --set full --clock-control none -k regex:"separable|axis_pass|cast" \
    -o gpurun_out/traffic/${c}_$f -f python tools/ncu_traffic.py run $c $f > gpurun_out/traffic/${c}_$f.log 2>&1
  touch gpurun_out/traffic/${c}_$f.csv
  echo "$c rc=$?"
done
python tools/ncu_traffic.py merge --out gpurun_out/ncu_summary_traffic.json gpurun_out/traffic/*.csv
rm -rf gpurun_out/traffic   # reports stay on the box (the merge-back limit is 64 MiB)
