mkdir -p gpurun_out
for c in A4 C; do python tools/s1_ab.py $c default:CURAST_LIB=tools/ab/w16.so 10 2 >> gpurun_out/late51_ab.jsonl 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "row_parallel" > gpurun_out/late51_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late51_tests.log
