mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for kv in "SR_FMG_CEXEC_STAGE=0" "SR_FMG_CEXEC_STAGE=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|coarse" gpurun_out/bd.log >> gpurun_out/sweep.log
done
