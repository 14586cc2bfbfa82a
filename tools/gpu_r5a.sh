# P27 bench line after the 27-point pass change; 27-point parity tests
mkdir -p gpurun_out
timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/r2_bench_p27_27pt.json 2> gpurun_out/r2_bench_p27.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "27" > gpurun_out/p27_pt2.log 2>&1; echo "rc=$?" >> gpurun_out/p27_pt2.log
