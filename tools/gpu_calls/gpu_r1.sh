set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_multirank.py -q -m gpu -p no:cacheprovider > gpurun_out/r1_newtests.log 2>&1
echo "newtests rc=$?" >> gpurun_out/r1_newtests.log
./tools/red_min_probe > gpurun_out/r1_red_probe.txt 2>&1
M=gpu__time_duration.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_s1_exact|k_stage2|k_stage3|k_clear" -c 12 --csv python tools/frame_once.py A4 2 > gpurun_out/r1_red_A4.csv 2> gpurun_out/r1_red_A4.err
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_s1_exact|k_stage2|k_stage3" -c 9 --csv python tools/frame_once.py C 2 > gpurun_out/r1_red_C.csv 2> gpurun_out/r1_red_C.err
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_red" -c 3 --csv ./tools/red_min_probe > gpurun_out/r1_red_probe.csv 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_gpu_configs.py --deselect tests/test_gpu_multirank.py > gpurun_out/r1_alltests.log 2>&1
echo "alltests rc=$?" >> gpurun_out/r1_alltests.log
