mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/breakdown.py > gpurun_out/breakdown.log 2>&1
timeout 600 python tools/breakdown.py --dtype f32 > gpurun_out/breakdown32.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
