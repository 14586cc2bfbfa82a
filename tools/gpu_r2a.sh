# round 2, first box run: GPU tests, smoke, bench, breakdowns (default and step kernels on
# levels 5-6)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python tools/breakdown.py > gpurun_out/bd_default.txt 2>&1
SR_FMG_FUSED_MIN_E=30 timeout 300 python tools/breakdown.py > gpurun_out/bd_min30.txt 2>&1
SR_FMG_FUSED_MIN_E=20 timeout 300 python tools/breakdown.py > gpurun_out/bd_min20.txt 2>&1
SR_FMG_CEXEC_PROF=1 timeout 300 python tools/cexec_prof.py > gpurun_out/cexec_prof.txt 2> gpurun_out/cexec_prof.err
