mkdir -p gpurun_out
rm -f gpurun_out/r13_ab.jsonl
for c in A B C D Dq; do python tools/s1_ab.py $c default 20 1 >> gpurun_out/r13_ab.jsonl 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_switches.py tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/r13_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r13_tests.log
