# flakiness check of the multi-rank tests
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_multirank.py -q -k "4x1x2-f32" 2>&1 | tail -1; done > gpurun_out/flaky.log 2>&1
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_multirank.py -q 2>&1 | tail -1; done >> gpurun_out/flaky.log 2>&1
