mkdir -p gpurun_out
: > gpurun_out/bench3.log
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | grep '^{' >> gpurun_out/bench3.log; done
for i in 1 2; do SR_FMG_TAU_FUSE=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | grep '^{' >> gpurun_out/bench3.log; done
