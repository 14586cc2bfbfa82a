mkdir -p gpurun_out
: > gpurun_out/sweep.log
for kv in "X=0" "X=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|k_cheb2" gpurun_out/bd.log >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd.log 2>&1
  grep -E "solve|k_cheb2" gpurun_out/bd.log >> gpurun_out/sweep.log
done
