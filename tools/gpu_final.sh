# round evidence: GPU suite, launch lists (fp64/fp32), full captures of the finest cheb2 pass and
# the fused FMG entry, bench lines (fp64 with cpu_baseline, fp32), in-graph breakdown
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_f64.csv python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1_launches_f32.csv python tools/ncu_solve.py --config C3 --dtype f32 --what solve --graph 0 > gpurun_out/ncu_list32.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r1_cheb_full -f python tools/ncu_solve.py --config C3 --what cheb --graph 0 > gpurun_out/ncu_cheb.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_pset1s --launch-skip 1 -c 1 -o gpurun_out/r1_pset_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_pset.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --dtype f32 --no-cpu-baseline > gpurun_out/bench_r1_f32.log 2>&1
timeout 600 python tools/breakdown.py > gpurun_out/breakdown_r1.log 2>&1
timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r1_p27.log 2>&1
timeout 600 python tools/breakdown.py --dtype f32 > gpurun_out/breakdown_r1_f32.log 2>&1
