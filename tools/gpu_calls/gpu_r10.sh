mkdir -p gpurun_out
python tools/s1_ab.py D default:CURAST_INSTANCED_KERNEL=1:CURAST_ILV=0 10 2 > gpurun_out/r10_ab_D.jsonl 2>&1
python tools/s1_ab.py A default:CURAST_ILV=1 30 1 > gpurun_out/r10_ab_A.jsonl 2>&1
python tools/s1_ab.py B default 30 1 > gpurun_out/r10_ab_B.jsonl 2>&1
python tools/s1_ab.py C default 30 1 > gpurun_out/r10_ab_C.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_switches.py tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r10_tests.log
