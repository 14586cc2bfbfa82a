timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "nonlinear or 27pt" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
