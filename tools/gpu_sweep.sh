mkdir -p gpurun_out
: > gpurun_out/sweep.log
for kv in "SR_FMG_CEXEC_TINY=512" "SR_FMG_CEXEC_TINY=4096" "SR_FMG_CEXEC_TINY=40000"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|coarse" gpurun_out/bd.log >> gpurun_out/sweep.log
done
