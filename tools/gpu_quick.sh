mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "x_shuffles" > gpurun_out/pytest_x.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_x.log
: > gpurun_out/sweep.log
for kv in "SR_FMG_RESTRICT_X=0" "SR_FMG_RESTRICT_X=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict" gpurun_out/bd.log >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict" gpurun_out/bd.log >> gpurun_out/sweep.log
done
