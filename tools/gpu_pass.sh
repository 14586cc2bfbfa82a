timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused_pass" > gpurun_out/pytest_pass.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pass.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode0.log 2>&1
SR_FMG_PASS_ENTRY=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode1.log 2>&1
SR_FMG_PASS_ENTRY=3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode3.log 2>&1
SR_FMG_PASS_ENTRY=4 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode4.log 2>&1
