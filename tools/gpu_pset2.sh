# pset.cu: GPU suite (incl. the new entry tests), breakdown, one full ncu capture of k_pset1s
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fmg_entry or fused" > gpurun_out/pytest_pset.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pset.log
timeout 600 python tools/breakdown.py > gpurun_out/breakdown.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_pset1s -c 1 -o gpurun_out/pset_full -f python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_pset.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_f64.csv python tools/ncu_solve.py --config C3 --what solve --graph 0 > gpurun_out/ncu_list.log 2>&1
