mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/resolve_ab.py B,A,A4,C $R/libR1.so:$R/libR2.so:$R/libR3.so:$R/libR4.so 20 > gpurun_out/r8_resolve_ab.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_resolve.py tests/test_gpu_debug_view.py -q -m gpu -p no:cacheprovider > gpurun_out/r8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r8_tests.log
