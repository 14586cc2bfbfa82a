timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e0.log 2>&1
SR_FMG_PASS_ENTRY=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e1.log 2>&1
SR_FMG_PASS_ENTRY=1 timeout 300 python tools/breakdown.py > gpurun_out/breakdown_e1.log 2>&1
