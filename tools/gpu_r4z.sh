# 27-point pass with shared in-plane row sums: parity (27-point tests), A/B on P27
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -k "27" > gpurun_out/p27_pt.log 2>&1; echo "rc=$?" >> gpurun_out/p27_pt.log
cp paper_1406_7808_b200/libsrfmg.so /tmp/new.so
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then cp ab/libsrfmg_base.so paper_1406_7808_b200/libsrfmg.so; else cp /tmp/new.so paper_1406_7808_b200/libsrfmg.so; fi
  echo "== $v"; timeout 300 python tools/breakdown.py --config P27 --stencil 27pt 2>&1 | head -6
done; done > gpurun_out/ab_p27.txt 2>&1
cp /tmp/new.so paper_1406_7808_b200/libsrfmg.so
