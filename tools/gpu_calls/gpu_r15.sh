mkdir -p gpurun_out
python tools/configs.py A B C D Bq Dq E200 A4 > gpurun_out/r15_configs.jsonl 2> gpurun_out/r15_configs.err
python tools/configs.py A C --check > gpurun_out/r15_configs_check.jsonl 2>> gpurun_out/r15_configs.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_s1_v2|k_s1_exact" -s 2 -c 2 -o gpurun_out/r15_B_full python tools/frame_once.py B 1 > gpurun_out/r15_ncu_B.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum
for c in B A4; do
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_resolve|k_downsample" -s 2 -c 2 --csv python tools/resolve_once.py $c > gpurun_out/r15_ncu_resolve_$c.csv 2> gpurun_out/r15_ncu_resolve_$c.err
done
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_s1|k_stage" -c 8 --csv python tools/frame_once.py D 1 > gpurun_out/r15_ncu_D.csv 2> gpurun_out/r15_ncu_D.err
