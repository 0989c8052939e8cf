mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT/build
python tools/s1_ab.py Bq CURAST_LIB=$R/libH.so:CURAST_LIB=$R/libN.so 20 2 > gpurun_out/r28_ab.jsonl 2>&1
python tools/s1_ab.py A CURAST_LIB=$R/libH.so 20 1 >> gpurun_out/r28_ab.jsonl 2>&1
python tools/s1_ab.py C CURAST_LIB=$R/libH.so 20 1 >> gpurun_out/r28_ab.jsonl 2>&1
