mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_switches.py tests/test_gpu_configs.py -x -q -m gpu -p no:cacheprovider > gpurun_out/r4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r4_tests.log
python tools/s1_ab.py B default 30 2 > gpurun_out/r4_ab_B.jsonl 2>&1
python tools/s1_ab.py D default:CURAST_ILV=0:CURAST_INSTANCED_KERNEL=1 10 1 > gpurun_out/r4_ab_D.jsonl 2>&1
python tools/s1_ab.py A default 30 1 > gpurun_out/r4_ab_A.jsonl 2>&1
python tools/s1_ab.py C default 30 1 > gpurun_out/r4_ab_C.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_s1" -c 2 --csv python tools/frame_once.py B 1 > gpurun_out/r4_ncu_B.csv 2> gpurun_out/r4_ncu_B.err
