mkdir -p gpurun_out
: > gpurun_out/sweep.log
for a in 0 7; do
  echo "== PSET_ALT=$a C5" >> gpurun_out/sweep.log
  SR_FMG_PSET_ALT=$a timeout 600 python tools/breakdown.py --config C5 > gpurun_out/bd.log 2>&1
  grep -E "solve|pass_entry" gpurun_out/bd.log >> gpurun_out/sweep.log
done
