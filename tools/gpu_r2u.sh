mkdir -p gpurun_out
for i in 1 2 3; do
SR_FMG_SYNC=1 timeout 60 python tools/single_debug.py 512,512,512 8 64 4 4 > gpurun_out/up_s3_$i.log 2>&1; echo "rc=$?" >> gpurun_out/up_s3_$i.log
done
SR_FMG_SYNC=1 timeout 60 python tools/single_debug.py 512,512,512 8 64 4 4 graph > gpurun_out/up_sg.log 2>&1; echo "rc=$?" >> gpurun_out/up_sg.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "up_pass or full_size_c3 or fp32" > gpurun_out/up_pt.log 2>&1; echo "rc=$?" >> gpurun_out/up_pt.log
timeout 300 python tools/breakdown.py > gpurun_out/bd_up64.txt 2>&1
SR_FMG_UP_FUSE=0 timeout 300 python tools/breakdown.py > gpurun_out/bd_noup64.txt 2>&1
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_up32.txt 2>&1
SR_FMG_UP_FUSE=0 timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_noup32.txt 2>&1
