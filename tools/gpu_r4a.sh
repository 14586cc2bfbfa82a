# session-2 re-entry check of HEAD: GPU suite, smoke, C3 bench lines (fp64, fp32), breakdown
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r4_bench_c3_f64.json 2> gpurun_out/r4_bench_c3_f64.err
timeout 600 python bench.py --steps 20 --warmup 5 --dtype f32 --no-cpu-baseline --no-accuracy > gpurun_out/r4_bench_c3_f32.json 2> gpurun_out/r4_bench_c3_f32.err
timeout 300 python tools/breakdown.py > gpurun_out/r4_breakdown_c3_f64.txt 2>&1
