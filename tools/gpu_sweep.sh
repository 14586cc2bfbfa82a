mkdir -p gpurun_out
: > gpurun_out/sweep.log
for a in 0 6 7 4; do
  echo "== ALT40=$a f64" >> gpurun_out/sweep.log
  SR_FMG_CHEB2_ALT40=$a timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|k_cheb2 .*l=7" gpurun_out/bd.log >> gpurun_out/sweep.log
done
