# wide coarse level fix: new parity tests, C5 K x S sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_coarse or sr_level_sweep or c5 or prolong" > gpurun_out/wide_pt.log 2>&1; echo "rc=$?" >> gpurun_out/wide_pt.log
timeout 1200 python tools/c5_sweep.py > gpurun_out/c5_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/c5_sweep.log
