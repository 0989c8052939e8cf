mkdir -p gpurun_out
python tools/s1_ab.py B default:CURAST_PIPE=0 20 3 > gpurun_out/r16_ab_B.jsonl 2>&1
python tools/s1_ab.py Bq default:CURAST_PIPE=0 10 2 > gpurun_out/r16_ab_Bq.jsonl 2>&1
python tools/s1_ab.py C default:CURAST_PIPE=0 10 2 > gpurun_out/r16_ab_C.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r16_tests.log
