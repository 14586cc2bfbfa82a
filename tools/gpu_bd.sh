timeout 600 python tools/breakdown.py > gpurun_out/breakdown.log 2>&1
