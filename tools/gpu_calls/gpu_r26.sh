mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libM4.so:CURAST_LIB=$R/libM5.so:CURAST_LIB=$R/libM6.so 20 2 > gpurun_out/r26_ab.jsonl 2>&1
