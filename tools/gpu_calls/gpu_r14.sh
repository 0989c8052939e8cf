mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libP0.so:CURAST_LIB=$R/libP1.so 30 3 > gpurun_out/r14_ab_B.jsonl 2>&1
python tools/s1_ab.py C CURAST_LIB=$R/libP0.so:CURAST_LIB=$R/libP1.so 30 1 > gpurun_out/r14_ab_C.jsonl 2>&1
