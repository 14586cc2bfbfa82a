mkdir -p gpurun_out
: > gpurun_out/sweep.log
timeout 900 env SR_FMG_PASS_RESTRICT=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "restriction or tau_fused or fmg_entry" > gpurun_out/pytest_pr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pr.log
for kv in "SR_FMG_PASS_RESTRICT=0" "SR_FMG_PASS_RESTRICT=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict" gpurun_out/bd.log >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict" gpurun_out/bd.log >> gpurun_out/sweep.log
done
