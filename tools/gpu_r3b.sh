# tiny-level runs of the coarse executor mirrored in shared memory: parity, multirank, per-op times, breakdowns
mkdir -p gpurun_out
SR_FMG_SYNC=1 timeout 120 python tools/single_debug.py 512,512,512 8 64 4 2 > gpurun_out/mi_sync.log 2>&1; echo "rc=$?" >> gpurun_out/mi_sync.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/mi_pt.log 2>&1; echo "rc=$?" >> gpurun_out/mi_pt.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -m gpu > gpurun_out/mi_mr.log 2>&1; echo "rc=$?" >> gpurun_out/mi_mr.log
timeout 120 python tools/cexec_prof.py > gpurun_out/mi_cexec.log 2> gpurun_out/mi_cexec.err
SR_FMG_CEXEC_MIRROR=0 timeout 120 python tools/cexec_prof.py > gpurun_out/mi0_cexec.log 2> gpurun_out/mi0_cexec.err
timeout 300 python tools/breakdown.py > gpurun_out/bd_mi64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_mi32.txt 2>&1
