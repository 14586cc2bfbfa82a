mkdir -p gpurun_out
for v in S T; do cp ab/lib_$v.so paper_1406_7808_b200/libsrfmg.so; echo "== $v"; timeout 120 python tools/f32check.py 2>&1 | tail -2; done > gpurun_out/pk_var.log
