timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c5_shapes or c4_two or host_async" --durations=5 > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
