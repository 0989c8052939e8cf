mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_multirank.py -q -x -m gpu -p no:cacheprovider -k "config_e" > gpurun_out/late82_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late82_tests.log
timeout 1500 python bench.py --mode E --steps 5 --warmup 3 --profile > gpurun_out/late82_E.log 2>&1; echo "rc=$?" >> gpurun_out/late82_E.log
timeout 1500 python bench.py --mode E --e-compressed --steps 5 --warmup 3 --profile > gpurun_out/late82_Eq.log 2>&1; echo "rc=$?" >> gpurun_out/late82_Eq.log
