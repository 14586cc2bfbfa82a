mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "thin or noncubic or C1" > gpurun_out/pytest_thin.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_thin.log
timeout 900 python tools/paper_tables.py > gpurun_out/paper_tables.log 2>&1; echo "rc=$?" >> gpurun_out/paper_tables.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2_f64.log 2> gpurun_out/bench_r2_f64.err
timeout 600 python bench.py --steps 20 --warmup 5 --dtype f32 --no-cpu-baseline > gpurun_out/bench_r2_f32.log 2> gpurun_out/bench_r2_f32.err
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_r2_f32.txt 2>&1
