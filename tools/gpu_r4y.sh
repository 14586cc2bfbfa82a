# coarse executor with 1024-thread CTAs (2-plane register batches) vs 512: bitwise check + A/B
mkdir -p gpurun_out
cp ab/lib_c1024.so paper_1406_7808_b200/libsrfmg.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "C1 or C2 or noncubic or thin or executor or coarse or kernel or dd-2x2x2 or full_size_c3_matches" > gpurun_out/c1024_pt.log 2>&1; echo "rc=$?" >> gpurun_out/c1024_pt.log
for rep in 1 2; do for v in base c1024; do
  if [ $v = base ]; then cp ab/libsrfmg_base.so paper_1406_7808_b200/libsrfmg.so; else cp ab/lib_c1024.so paper_1406_7808_b200/libsrfmg.so; fi
  echo "== $v f64"; timeout 300 python tools/breakdown.py 2>&1 | grep -E "solve|k_coarse"
  echo "== $v f32"; timeout 300 python tools/breakdown.py --dtype f32 2>&1 | grep -E "solve|k_coarse"
done; done > gpurun_out/ab_c1024.txt 2>&1
