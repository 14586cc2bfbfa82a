mkdir -p gpurun_out
: > gpurun_out/sweep.log
for a in 0 4; do for dt in f32 f64; do
  echo "== PSET_ALT=$a $dt" >> gpurun_out/sweep.log
  SR_FMG_PSET_ALT=$a timeout 300 python tools/breakdown.py --dtype $dt > gpurun_out/bd.log 2>&1
  grep -E "solve|pass_entry" gpurun_out/bd.log >> gpurun_out/sweep.log
done; done
