# round-2 final evidence (session 2, profiling-ring bench): GPU suite, smoke, bench lines, breakdowns, ncu launch lists
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_f64.json 2> gpurun_out/r2_bench_c3_f64.err
timeout 600 python bench.py --steps 20 --warmup 5 --dtype f32 --no-cpu-baseline > gpurun_out/r2_bench_c3_f32.json 2> gpurun_out/r2_bench_c3_f32.err
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2_bench_c5_f64.json 2> gpurun_out/r2_bench_c5_f64.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1
timeout 300 python tools/breakdown.py > gpurun_out/r2_breakdown_c3_f64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/r2_breakdown_c3_f32.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3_f64.csv python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3_f32.csv python tools/ncu_solve.py --config C3 --dtype f32 --what solve --graph 0 > gpurun_out/ncu_list32.log 2>&1
