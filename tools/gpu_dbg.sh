export SR_FMG_FORCE_FUSED=1
timeout 300 python tools/dbg_pass.py 1 4 512 > gpurun_out/dbgA.log 2>&1
DBG_REPS=5 timeout 300 python tools/dbg_pass.py 1 4 512 > gpurun_out/dbgB.log 2>&1
DBG_GRAPH=1 timeout 300 python tools/dbg_pass.py 1 4 512 > gpurun_out/dbgC.log 2>&1
DBG_GRAPH=1 DBG_REPS=5 timeout 300 python tools/dbg_pass.py 1 4 512 > gpurun_out/dbgD.log 2>&1
DBG_GRAPH=1 DBG_REPS=5 timeout 300 python tools/dbg_pass.py 1 3 128 ref > gpurun_out/dbgE.log 2>&1
DBG_GRAPH=1 DBG_REPS=5 SR_FMG_PASS_MAXPY=40 timeout 300 python tools/dbg_pass.py 1 4 512 > gpurun_out/dbgF.log 2>&1
