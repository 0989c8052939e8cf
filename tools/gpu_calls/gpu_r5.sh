mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libA.so:CURAST_LIB=$R/libB.so:CURAST_LIB=$R/libC.so 30 3 > gpurun_out/r5_ab_B.jsonl 2>&1
for L in A B C; do
CURAST_LIB=$R/lib$L.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_s1_v2" -c 1 --csv python tools/frame_once.py B 1 > gpurun_out/r5_ncu_$L.csv 2> gpurun_out/r5_ncu_$L.err
done
