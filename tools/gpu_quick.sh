mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/breakdown.py > gpurun_out/bd_c3.log 2>&1
timeout 600 python tools/breakdown.py --config P27 --stencil 27pt > gpurun_out/bd_p27.log 2>&1
timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p27.log 2>&1
