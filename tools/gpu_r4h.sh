# coarse executor per-operation cycles (C3 fp64)
mkdir -p gpurun_out
timeout 300 python tools/cexec_prof.py > gpurun_out/cexec_prof.log 2>&1; echo "rc=$?" >> gpurun_out/cexec_prof.log
