# lean degree-2 pass: parity subset + A/B breakdown
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or full_size_c3 or smoke or C1 or C2" > gpurun_out/pytest_lean.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lean.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_lean.txt 2>&1
SR_FMG_CHEB_LEAN=0 timeout 300 python tools/breakdown.py > gpurun_out/bd_nolean.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_lean32.txt 2>&1
SR_FMG_CHEB_LEAN=0 timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_nolean32.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_lean.log 2>&1
