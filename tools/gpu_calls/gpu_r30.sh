mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libX1.so:CURAST_LIB=$R/libX2.so 20 2 > gpurun_out/r30_ab.jsonl 2>&1
python tools/s1_ab.py D CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libX1.so 10 1 >> gpurun_out/r30_ab.jsonl 2>&1
