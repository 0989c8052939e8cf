mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/late89_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late89_tests.log
