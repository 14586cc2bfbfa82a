mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -k "27pt_and_nonlinear" > gpurun_out/ops_mr.log 2>&1; echo "rc=$?" >> gpurun_out/ops_mr.log
