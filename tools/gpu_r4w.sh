# packed fp32 pass at 4 CTAs/SM (96 registers, small spills) vs 3 (126 registers): A/B
mkdir -p gpurun_out
cp paper_1406_7808_b200/libsrfmg.so /tmp/keep.so
for rep in 1 2; do for v in base m4; do
  if [ $v = base ]; then cp ab/libsrfmg_base.so paper_1406_7808_b200/libsrfmg.so; else cp ab/lib_m4.so paper_1406_7808_b200/libsrfmg.so; fi
  echo "== $v"; timeout 300 python tools/breakdown.py --dtype f32 2>&1 | grep -E "solve|k_cheb2 +l=8"
done; done > gpurun_out/ab_m4.txt 2>&1
