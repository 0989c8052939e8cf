mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_s1" -c 2 --csv python tools/frame_once.py B 1 > gpurun_out/r13_ncu_B_def.csv 2> gpurun_out/r13_def.err
CURAST_LIB=tools/ab/pk.so CURAST_F32_PACKED=1 timeout 600 ncu --metrics $M --clock-control none -k regex:"k_s1" -c 2 --csv python tools/frame_once.py B 1 > gpurun_out/r13_ncu_B_pk.csv 2> gpurun_out/r13_pk.err
