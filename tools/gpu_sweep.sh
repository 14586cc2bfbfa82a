mkdir -p gpurun_out
: > gpurun_out/sweep.log
for kv in "SR_FMG_SEGEXEC=0" "SR_FMG_SEG_NB=2" "SR_FMG_SEG_NB=3"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  cat gpurun_out/bd.log >> gpurun_out/sweep.log
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
