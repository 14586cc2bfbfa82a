mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "27pt" > gpurun_out/pytest_27.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_27.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.log
for kv in "SR_FMG_TAU_FUSE=0" "SR_FMG_TAU_FUSE=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 600 python tools/breakdown.py --config P27 --stencil 27pt > gpurun_out/bd.log 2>&1
  grep -E "solve|tau|k_cheb2" gpurun_out/bd.log >> gpurun_out/sweep.log
done
