mkdir -p gpurun_out
timeout 40 python tools/single_debug.py 64,32,32 5 16 2 > gpurun_out/sd_a.log 2>&1; echo "rc=$?" >> gpurun_out/sd_a.log
timeout 60 python tools/dd_debug.py --dump 45 > gpurun_out/dd_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dd_dbg.log
timeout 700 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_multirank.py > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_r2k.txt 2>&1
