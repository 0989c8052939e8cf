mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libP0.so:CURAST_LIB=$R/libP1.so:CURAST_LIB=$R/libP2.so:CURAST_LIB=$R/libP4.so 20 2 > gpurun_out/r27_ab.jsonl 2>&1
