python tools/lu_probe.py 8192 16384 32768 > gpurun_out/lu_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lu16k_launches.csv python tools/profile_run.py lu 16384 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/lu16k_launches.csv > gpurun_out/lu16k_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:colstream_mv -s 2 -c 1 -o gpurun_out/gemv32k_full python tools/profile_run.py gemv 32768 > gpurun_out/gemv32k_ncu.log 2>&1
ncu -i gpurun_out/gemv32k_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/gemv32k_raw.csv 2>&1
cat gpurun_out/lu_probe.txt gpurun_out/lu16k_summary.txt gpurun_out/gemv32k_raw.csv
