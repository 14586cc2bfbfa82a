mkdir -p gpurun_out
for alt in 0 2 3; do for dt in f64 f32; do
  echo "alt=$alt $dt" >> gpurun_out/pset_sweep.log
  SR_FMG_PSET_ALT=$alt timeout 300 python tools/breakdown.py --dtype $dt > gpurun_out/bd.log 2>&1
  grep -E "^solve|pass_entry" gpurun_out/bd.log >> gpurun_out/pset_sweep.log
done; done
for alt in 2 3; do SR_FMG_PSET_ALT=$alt timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fmg_entry" >> gpurun_out/pytest_pset.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pset.log; done
