mkdir -p gpurun_out
for mb in 5 6; do SR_FMG_RESTRICT_MINB=$mb timeout 200 python tools/breakdown.py > gpurun_out/bdo_mb$mb.txt 2>&1; done
timeout 200 python tools/breakdown.py > gpurun_out/bdo_base.txt 2>&1
