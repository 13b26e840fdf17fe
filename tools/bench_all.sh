#!/bin/bash
# all bench configs on one GPU + launch list + ncu captures of the top kernels
# usage (repo root, on the GPU box): tools/bench_all.sh   -> gpurun_out/round/
mkdir -p gpurun_out/round
for c in c2 c1 c3-9 c3-15 c3-21 c3-31 c4 c5 c6-143 c6-245 c6-450 c6-921; do
  timeout 900 python bench.py --config $c > gpurun_out/round/bench_$c.json 2> gpurun_out/round/bench_$c.err
  echo "$c rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/round/bench_$c.json')); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"
done
timeout 900 python bench.py --impl reference > gpurun_out/round/bench_reference_c2.json 2> gpurun_out/round/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/round/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/round/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:separable_kernel -c 1 -o gpurun_out/round/sep_c2 python tools/prof_sep.py 16 > gpurun_out/round/ncu_sep.log 2>&1; echo "sep rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dct16_kernel -c 1 -o gpurun_out/round/dct16 python tools/time_dct.py > gpurun_out/round/ncu_dct.log 2>&1; echo "dct rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:axis_pass_kernel -c 2 -o gpurun_out/round/apass python tools/time_two_pass.py > gpurun_out/round/ncu_apass.log 2>&1; echo "apass rc=$?"
