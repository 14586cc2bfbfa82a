mkdir -p gpurun_out
timeout 900 python tools/paper_tables.py > gpurun_out/paper_tables.log 2>&1; echo "rc=$?" >> gpurun_out/paper_tables.log
timeout 900 python tools/accuracy_table.py > gpurun_out/accuracy.log 2>&1; echo "rc=$?" >> gpurun_out/accuracy.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "large_segments or fused_and_step or fp32" > gpurun_out/pytest_large.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_large.log
timeout 300 python tools/breakdown.py --dtype f32 > gpurun_out/bd_f32_new.txt 2>&1
