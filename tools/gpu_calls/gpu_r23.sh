mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_s1" -s 2 -c 2 --csv python tools/frame_once.py D 1 > gpurun_out/r23_ncu_D.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_s1" -s 2 -c 2 --csv python tools/frame_once.py Bq 1 > gpurun_out/r23_ncu_Bq.csv 2>&1
