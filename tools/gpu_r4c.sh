# debug: idle at T mismatch under variations; K = 0 after the zT2 fix
mkdir -p gpurun_out
A="--n 64,64,64 --M 5 --seg 8 --J 2 --K 2 --pgrid 2,1,1 --dtype f64 --dd_min 0 --idle 1"
for v in "SR_FMG_CEXEC=0" "SR_FMG_FUSED=0" "SR_FMG_CEXEC=0 SR_FMG_FUSED=0" "SR_FMG_SYNC=1"; do
  echo "== $v" >> gpurun_out/dbg_var.log
  env $v timeout 120 python tools/dd_debug.py $A 2>&1 | grep "bitwise" >> gpurun_out/dbg_var.log
done
timeout 120 python tools/dd_debug.py --n 64,64,64 --M 5 --seg 0 --J 0 --K 0 --pgrid 2,1,1 --dtype f64 --dd_min 8 > gpurun_out/dbg_k0.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_k0.log
