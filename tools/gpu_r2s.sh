# fused up pass: parity subset, breakdown A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or full_size_c3 or C1 or C2 or C3 or noncubic or thin or entry or tau or large" > gpurun_out/pytest_up.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_up.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr_up.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr_up.log
timeout 200 python tools/breakdown.py > gpurun_out/bd_up64.txt 2>&1
SR_FMG_UP_FUSE=0 timeout 200 python tools/breakdown.py > gpurun_out/bd_noup64.txt 2>&1
timeout 200 python tools/breakdown.py --dtype f32 > gpurun_out/bd_up32.txt 2>&1
SR_FMG_UP_FUSE=0 timeout 200 python tools/breakdown.py --dtype f32 > gpurun_out/bd_noup32.txt 2>&1
