timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "vsolve or mbs" > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 900 python tools/compare_solvers.py > gpurun_out/solver_comparison.json 2> gpurun_out/solver_comparison.err
