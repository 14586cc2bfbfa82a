# idle coarse grid + conventional distributed FMG (K = 0): multi-rank GPU tests (host store)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -k idle_and > gpurun_out/mr.log 2>&1; echo "rc=$?" >> gpurun_out/mr.log
