mkdir -p gpurun_out
: > gpurun_out/sweep.log
for kv in "SR_FMG_COL_TARGET=800000" "SR_FMG_COL_TARGET=400000" "SR_FMG_COL_TARGET=1600000" "SR_FMG_COL_TARGET=1600000 SR_FMG_COL_MINZ=2"; do
  echo "== $kv f32" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict .*l=[78]" gpurun_out/bd.log >> gpurun_out/sweep.log
done
