# DD path: multirank threaded tests, then the whole GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
