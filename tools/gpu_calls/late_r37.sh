mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "forcing" > gpurun_out/late37_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late37_tests.log
