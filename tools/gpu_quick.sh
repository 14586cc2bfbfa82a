mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "S128 or C5 or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/breakdown.py --config C5 > gpurun_out/bd_c5.log 2>&1
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
