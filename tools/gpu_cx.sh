SR_FMG_CEXEC_PROF=1 timeout 300 python tools/dbg_pass.py 0 4 512 > gpurun_out/cexec_prof.log 2>&1
