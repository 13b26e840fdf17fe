#!/bin/bash
# Round-end evidence on one GPU box (repo root):
#   bench lines of every config, the c2 timed-region launch list (NVTX-filtered),
#   ncu --set full of each config's kernels (DRAM traffic per frame -> bench's
#   roofline.traffic), and per-kernel summaries of the c2 / c1 / c4 kernels.
# Output: gpurun_out/r02/ (summaries only; the .ncu-rep files stay on the box
# except the three kernel captures).
set -u
R=${R:-r02}
O=gpurun_out/$R
mkdir -p $O/traffic
CFGS=${CFGS:-"c2 c1 c3-9 c3-15 c3-21 c3-31 c4 c5 c6-143 c6-245 c6-450 c6-921"}
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-200} --warmup 5 > $O/bench_$c.json 2> $O/bench_$c.err
  echo "$c rc=$? $(python -c "import json; d=json.load(open('$O/bench_$c.json')); print(d['value'], d['roofline']['frac'], d['sustained']['roofline_frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_c2.json 2> $O/bench_reference.err; echo "reference rc=$?"
# the default bench command's timed region only (NVTX range bench.timed)
timeout 900 ncu --nvtx --nvtx-include "bench.timed/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $O/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > $O/launches_c2.log 2>&1; echo "launch list rc=$?"
# per-config DRAM traffic (one pipeline call, cold cache)
for c in $CFGS; do
  f=4; [ "${c%%-*}" = "c3" ] && f=1; [ "$c" = "c2" ] && f=16; [ "$c" = "c1" ] && f=16
  timeout 900 ncu --set full --clock-control none -k regex:"separable|axis_pass|cast|dct16" \
    -o $O/traffic/${c}_$f -f python tools/ncu_traffic.py run $c $f > $O/traffic/${c}_$f.log 2>&1
  touch $O/traffic/${c}_$f.csv
  echo "traffic $c rc=$?"
done
cp profiles/ncu_summary.json $O/ncu_summary.json
python tools/ncu_traffic.py merge --out $O/ncu_summary.json $O/traffic/*.csv
# kernel captures with source (kept: read them with tools/ncu_lines.py)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:separable_kernel -c 1 \
  -o $O/sep_c2 -f python tools/prof_sep.py 16 > $O/ncu_sep.log 2>&1; echo "sep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:separable_f32 -c 1 \
  -o $O/f32_c1 -f python tools/prof_f32.py > $O/ncu_f32.log 2>&1; echo "f32 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dct16_kernel -c 1 \
  -o $O/dct_c4 -f python tools/time_dct.py 16 > $O/ncu_dct.log 2>&1; echo "dct rc=$?"
python tools/ncu_summary.py $O/sep_c2.ncu-rep $O/launches_c2.csv $O/ncu_separable_c2 16
python tools/ncu_summary.py $O/f32_c1.ncu-rep - $O/ncu_f32_c1 16 $((3 * 1080 * 1920 * 4 + 3 * 540 * 960 * 4))
python tools/ncu_summary.py $O/dct_c4.ncu-rep - $O/ncu_dct16_c4 16 $((3 * 2160 * 3840 * 4))
rm -rf $O/traffic
