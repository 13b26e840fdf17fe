cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ap
timeout 600 ncu --set full --clock-control none --import-source on -k regex:axis_pass -c 2 -o gpurun_out/ap/apass_921 -f python tools/apass_split.py 921 > gpurun_out/ap/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/ap/apass_921.ncu-rep - gpurun_out/ap/ncu_axis_pass_921 48 $((2048 * 2048 * 2 + 921 * 921 * 2)) 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_smem_poison.py -q 2>&1 | tail -2
