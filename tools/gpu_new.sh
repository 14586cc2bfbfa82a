timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p27.log 2>&1
timeout 600 python bench.py --config P27 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p7.log 2>&1
timeout 600 python tools/breakdown.py --config P27 > gpurun_out/bd_p27_7.log 2>&1
timeout 600 python tools/breakdown.py --config P27 --stencil 27pt > gpurun_out/bd_p27_27.log 2>&1
