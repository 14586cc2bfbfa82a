mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank.py -m gpu -q > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
