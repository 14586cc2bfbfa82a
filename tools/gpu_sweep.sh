mkdir -p gpurun_out
: > gpurun_out/sweep.log
for a in 1 2 4 5 9; do
  echo "== ALT=$a" >> gpurun_out/sweep.log
  SR_FMG_CHEB2_ALT=$a timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|k_cheb2 .*l=8" gpurun_out/bd.log >> gpurun_out/sweep.log
done
