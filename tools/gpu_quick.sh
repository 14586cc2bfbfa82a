mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "27pt" > gpurun_out/pytest_27.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_27.log
timeout 600 python tools/breakdown.py --config P27 --stencil 27pt > gpurun_out/bd.log 2>&1
timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p27.log 2>&1
