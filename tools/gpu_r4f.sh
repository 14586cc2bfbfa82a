mkdir -p gpurun_out
for v in pack scal; do
  cp build/lib_$v.so paper_1406_7808_b200/libsrfmg.so
  echo "== $v"; timeout 300 python tools/pack_debug.py 2>&1 | grep -v "^  seg"
done > gpurun_out/pack_debug2.log
