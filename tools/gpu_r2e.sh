# DD fix + segment-resident passes: multirank (short), parity subset, breakdowns
mkdir -p gpurun_out
SR_FMG_SYNC=0 timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mr.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or full_size_c3 or C1 or C2 or kernel or tau or entry" > gpurun_out/pytest_seg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_seg.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_seg.txt 2>&1
SR_FMG_SEG=0 timeout 300 python tools/breakdown.py > gpurun_out/bd_noseg.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-accuracy > gpurun_out/bench_seg.log 2>&1
