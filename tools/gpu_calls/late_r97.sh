mkdir -p gpurun_out
python tools/resolve_ab.py B,A,A4,C paper_2604_21749_b200/libcurast_b200.so:tools/ab/base.so 20 > gpurun_out/late97_resolve_ab.jsonl 2>&1
python tools/resolve_ab.py B,C tools/ab/base.so:paper_2604_21749_b200/libcurast_b200.so 20 >> gpurun_out/late97_resolve_ab.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_resolve.py tests/test_gpu_debug_view.py -q -x -m gpu -p no:cacheprovider > gpurun_out/late97_tests.log 2>&1; echo "rc=$?" >> gpurun_out/late97_tests.log
