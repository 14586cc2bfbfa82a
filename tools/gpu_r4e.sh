mkdir -p gpurun_out
timeout 300 python tools/pack_debug.py > gpurun_out/pack_debug.log 2>&1; echo "rc=$?" >> gpurun_out/pack_debug.log
