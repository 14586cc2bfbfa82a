mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tau_fused" > gpurun_out/pytest_tau.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tau.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.log
for kv in "SR_FMG_TAU_FUSE=0" "SR_FMG_TAU_FUSE=1"; do
  echo "== $kv" >> gpurun_out/sweep.log
  env $kv timeout 300 python tools/breakdown.py > gpurun_out/bd.log 2>&1
  grep -E "solve|tau|k_cheb2" gpurun_out/bd.log >> gpurun_out/sweep.log
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
