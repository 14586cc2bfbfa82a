timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused_pass" > gpurun_out/pytest_pass.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pass.log
for m in 1 3 4; do SR_FMG_PASS=$m timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mode$m.log 2>&1; done
SR_FMG_PASS=1 timeout 600 python tools/breakdown.py > gpurun_out/breakdown_p1.log 2>&1
