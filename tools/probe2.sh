timeout 600 python -m pytest tests/test_gpu_direct.py tests/test_gpu_ops.py -x -q > gpurun_out/p2_pytest.log 2>&1; tail -3 gpurun_out/p2_pytest.log
python tools/lu_probe.py 16384 32768 > gpurun_out/lu_probe2.txt 2>&1; cat gpurun_out/lu_probe2.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu16k_launches2.csv python tools/profile_run.py lu 16384 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/lu16k_launches2.csv
