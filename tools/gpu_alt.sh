for a in 1 7 8 9; do SR_FMG_CHEB2_ALT=$a timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_alt64_$a.log 2>&1; done
