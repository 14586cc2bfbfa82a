for e in 0 15 23; do SR_FMG_FUSED_MIN_E=$e timeout 300 python tools/breakdown.py > gpurun_out/bd_mine_$e.log 2>&1; done
