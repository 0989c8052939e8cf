mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py B CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libV.so 20 3 > gpurun_out/r29_ab.jsonl 2>&1
python tools/s1_ab.py A CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libV.so 20 1 >> gpurun_out/r29_ab.jsonl 2>&1
