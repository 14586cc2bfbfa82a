mkdir -p gpurun_out
: > gpurun_out/sweep.log
for kv in "SR_FMG_CHEB2_ALT40=4" "SR_FMG_CHEB2_ALT40=5" "SR_FMG_CHEB2_ALT40=4 SR_FMG_CHEB2_ALT24=3"; do
  echo "== $kv f32" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|k_cheb2 .*l=[67]" gpurun_out/bd.log >> gpurun_out/sweep.log
done
