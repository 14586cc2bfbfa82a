mkdir -p gpurun_out
: > gpurun_out/sweep.log
for b in 18 10 13 24 38; do
  echo "== PROLONG_BH=$b f64" >> gpurun_out/sweep.log
  SR_FMG_PROLONG_BH=$b timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|prolong" gpurun_out/bd.log >> gpurun_out/sweep.log
done
