mkdir -p gpurun_out
python tools/s1_ab.py D default:CURAST_INSTANCED_KERNEL=1 10 2 > gpurun_out/r9_ab_D.jsonl 2>&1
python tools/s1_ab.py Dq default 10 1 > gpurun_out/r9_ab_Dq.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_switches.py tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "instanc or lantern or route or golden or config_d or dq" > gpurun_out/r9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r9_tests.log
CURAST_INSTANCED_KERNEL=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none -k regex:"k_s1" -c 2 --csv python tools/frame_once.py D 1 > gpurun_out/r9_ncu_D.csv 2> gpurun_out/r9_ncu_D.err
