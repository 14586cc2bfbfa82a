mkdir -p gpurun_out
run() { name=$1; shift; SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 45 python tools/dd_debug.py --dump 30 "$@" > gpurun_out/dd_$name.log 2>&1; echo "rc=$?" >> gpurun_out/dd_$name.log; }
run a_nodd --dd_min 1048576
run b_2x1 --n 64,32,32 --pgrid 2,1,1
run c_4x1_big --n 256,64,64 --M 6 --seg 32 --pgrid 4,1,1 --dtype f64
run d_4x1_dd4 --dd_min 4
run e_1x4 --n 32,128,32 --pgrid 1,4,1
