# 27-point interior fast path: bitwise vs the previous build, 27-point tests, A/B on P27
mkdir -p gpurun_out
cp paper_1406_7808_b200/libsrfmg.so /tmp/new.so
cp ab/libsrfmg_base.so paper_1406_7808_b200/libsrfmg.so; timeout 120 python tools/p27_dump.py /tmp/u_base.npy
cp /tmp/new.so paper_1406_7808_b200/libsrfmg.so; timeout 120 python tools/p27_dump.py /tmp/u_new.npy
python -c "import numpy as np; a=np.load('/tmp/u_base.npy'); b=np.load('/tmp/u_new.npy'); print('bitwise', np.array_equal(a,b), float(np.abs(a-b).max()))" > gpurun_out/p27i_bitwise.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -k "27" > gpurun_out/p27i_pt.log 2>&1; echo "rc=$?" >> gpurun_out/p27i_pt.log
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then cp ab/libsrfmg_base.so paper_1406_7808_b200/libsrfmg.so; else cp /tmp/new.so paper_1406_7808_b200/libsrfmg.so; fi
  echo "== $v"; timeout 300 python tools/breakdown.py --config P27 --stencil 27pt 2>&1 | head -4
done; done > gpurun_out/ab_p27i.txt 2>&1
cp /tmp/new.so paper_1406_7808_b200/libsrfmg.so
