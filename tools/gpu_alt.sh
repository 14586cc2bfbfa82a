for a in 0 1 2; do SR_FMG_CHEB2_ALT40=$a timeout 300 python tools/breakdown.py > gpurun_out/bd_a40_$a.log 2>&1; done
for a in 1 2; do SR_FMG_CHEB2_ALT24=$a timeout 300 python tools/breakdown.py > gpurun_out/bd_a24_$a.log 2>&1; done
