mkdir -p gpurun_out
python tools/s1_ab.py B default 30 2 > gpurun_out/r2_ab_B.jsonl 2>&1
python tools/s1_ab.py A default 30 1 > gpurun_out/r2_ab_A.jsonl 2>&1
python tools/s1_ab.py C default 30 1 > gpurun_out/r2_ab_C.jsonl 2>&1
for m in v2 v2f; do
CURAST_S1=$m timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio --clock-control none -k regex:"k_s1" -c 4 --csv python tools/frame_once.py B 1 > gpurun_out/r2_ncu_$m.csv 2> gpurun_out/r2_ncu_$m.err
done
