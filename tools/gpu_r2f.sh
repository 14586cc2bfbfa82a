# seg race fix + MLP, executor residency, DD f32 hang localisation
mkdir -p gpurun_out
SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 120 python -X faulthandler -m pytest tests/test_gpu_multirank.py -q -x -k "dd-4x1x1-f32-0" > gpurun_out/pytest_ddf32.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ddf32.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or full_size_c3 or C1 or C2 or kernel or tau or entry" > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_seg.txt 2>&1
SR_FMG_SEG=0 timeout 300 python tools/breakdown.py > gpurun_out/bd_noseg.txt 2>&1
SR_FMG_CEXEC_RES=0 timeout 300 python tools/breakdown.py > gpurun_out/bd_nores.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_seg.log 2>&1
