mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "row_parallel" > gpurun_out/late54_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late54_tests.log
