# fused up pass (fixed coarse staging): quick solve first, then parity, multirank, breakdowns
mkdir -p gpurun_out
timeout 60 python tools/single_debug.py 512,512,512 8 64 4 > gpurun_out/up_quick.log 2>&1; echo "rc=$?" >> gpurun_out/up_quick.log
if grep -q "done True" gpurun_out/up_quick.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "up_pass or full_size_c3 or C1 or C2 or C3 or noncubic or thin or entry or large" > gpurun_out/pytest_up.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_up.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr_up.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr_up.log
timeout 200 python tools/breakdown.py > gpurun_out/bd_up64.txt 2>&1
timeout 200 python tools/breakdown.py --dtype f32 > gpurun_out/bd_up32.txt 2>&1
fi
