# full GPU suite after making the fused up pass opt-in
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2x.log
