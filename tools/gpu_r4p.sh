# profiling ring: test, bench (new timed loop), breakdown for comparison
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "profiling_ring or up_pass_correction_and_smoothing" > gpurun_out/ring_pt.log 2>&1; echo "rc=$?" >> gpurun_out/ring_pt.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-accuracy > gpurun_out/ring_bench.json 2> gpurun_out/ring_bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-accuracy --dtype f32 > gpurun_out/ring_bench32.json 2>> gpurun_out/ring_bench.err
timeout 300 python tools/breakdown.py 2>&1 | head -3 > gpurun_out/ring_bd.txt
