mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "row_parallel or forcing" > gpurun_out/late48_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late48_tests.log
python tools/s1_ab.py C default 20 2 > gpurun_out/late48_ab.jsonl 2>&1
python tools/s1_ab.py B default 20 2 >> gpurun_out/late48_ab.jsonl 2>&1
python tools/s1_ab.py A default 20 1 >> gpurun_out/late48_ab.jsonl 2>&1
