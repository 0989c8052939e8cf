mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
rm -f gpurun_out/r22_ab.jsonl
for c in B C A; do python tools/s1_ab.py $c CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libN.so 20 2 >> gpurun_out/r22_ab.jsonl 2>&1; done
CURAST_LIB=$R/libN.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_s1_v2" -s 1 -c 1 --csv python tools/frame_once.py B 1 > gpurun_out/r22_ncu.csv 2>&1
