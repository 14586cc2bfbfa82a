mkdir -p gpurun_out
SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 100 python tools/dd_debug.py --dump 60 > gpurun_out/dd_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dd_dbg.log
SR_FMG_SEG=0 SR_FMG_TRACE=1 SR_FMG_SYNC=1 timeout 100 python tools/dd_debug.py --dump 60 > gpurun_out/dd_dbg_noseg.log 2>&1; echo "rc=$?" >> gpurun_out/dd_dbg_noseg.log
timeout 100 python tools/dd_debug.py --dtype f64 --dump 60 > gpurun_out/dd_dbg64.log 2>&1; echo "rc=$?" >> gpurun_out/dd_dbg64.log
for t in 400000 800000 1600000; do SR_FMG_SEG=0 SR_FMG_CEXEC_RES=0 SR_FMG_COL_TARGET=$t timeout 300 python tools/breakdown.py > gpurun_out/bd_col$t.txt 2>&1; done
