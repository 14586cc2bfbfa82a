mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.log
for kv in "SR_FMG_RESTRICT_PYR=0" "SR_FMG_RESTRICT_PYR=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 600 python tools/breakdown.py --config P27 --stencil 27pt > gpurun_out/bd.log 2>&1
  grep -E "solve|restrict" gpurun_out/bd.log >> gpurun_out/sweep.log
done
timeout 600 python bench.py --config P27 --stencil 27pt --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p27.log 2>&1
