mkdir -p gpurun_out
SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 40 python tools/single_debug.py 64,32,32 5 16 2 > gpurun_out/sd_a.log 2>&1; echo "rc=$?" >> gpurun_out/sd_a.log
SR_FMG_CEXEC_ONE=1 SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 40 python tools/single_debug.py 64,32,32 5 16 2 > gpurun_out/sd_one.log 2>&1; echo "rc=$?" >> gpurun_out/sd_one.log
